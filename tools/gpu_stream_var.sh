cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
run() { timeout 300 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bv.json 2>gpurun_out/bv.err; python -c "
import json,sys; d=json.load(open('gpurun_out/bv.json')); print(sys.argv[1], round(d['value']), d['clocks']['sm_mhz'], d['clocks']['reasons'])" "$1" 2>/dev/null || echo "$1 FAILED"; }
for lib in i0 i200 i1000 i0 i200 i1000 i0 i200; do
  cp tools/variants/lib_$lib.so paper_2105_05879_b200/libfst_b200.so; run $lib
done
cp tools/variants/lib_i0.so paper_2105_05879_b200/libfst_b200.so
