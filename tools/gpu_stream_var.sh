cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
run() { timeout 300 python bench.py --config $1 --steps $2 --warmup 3 --no-cpu --no-e2e > gpurun_out/bv.json 2>gpurun_out/bv.err; python -c "
import json,sys; d=json.load(open('gpurun_out/bv.json')); print(sys.argv[1], round(d['value']), d['clocks']['sm_mhz'])" "$3 config $1" 2>/dev/null || echo "$3 FAILED"; }
for lib in cw8r64 cw6r64 cw8r128 cw6r128 cw8r64 cw6r64 cw8r128 cw6r128; do
  cp tools/variants/lib_$lib.so paper_2105_05879_b200/libfst_b200.so
  run 3 3 $lib
done
cp tools/variants/lib_cw8r64.so paper_2105_05879_b200/libfst_b200.so
