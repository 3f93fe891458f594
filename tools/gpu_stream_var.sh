cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
run() { timeout 300 python bench.py --config $1 --steps $2 --warmup 3 --no-cpu --no-e2e > gpurun_out/bv.json 2>gpurun_out/bv.err; python -c "
import json,sys; d=json.load(open('gpurun_out/bv.json')); print(sys.argv[1], round(d['value']), d['clocks']['sm_mhz'])" "$3 config $1"; }
for lib in dbg nodbg dbg nodbg; do
  cp tools/variants/lib_$lib.so paper_2105_05879_b200/libfst_b200.so
  run 3 3 $lib; run 2 10 $lib
done
cp tools/variants/lib_nodbg.so paper_2105_05879_b200/libfst_b200.so
