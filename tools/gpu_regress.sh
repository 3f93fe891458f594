cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
run() { timeout 300 python bench.py --config $1 --steps $3 --warmup 3 --no-cpu --no-e2e > gpurun_out/rg.json 2>gpurun_out/rg.err; python -c "
import json,sys; d=json.load(open('gpurun_out/rg.json')); print(sys.argv[1], round(d['value']), d['clocks']['sm_mhz'])" "$2 config $1" 2>/dev/null || echo "$2 config $1 FAILED"; }
for lib in r6 cur fix r6 fix; do
  cp tools/variants/lib_$lib.so paper_2105_05879_b200/libfst_b200.so
  run 2 $lib 10; run 1 $lib 10; run 3 $lib 3
done
cp tools/variants/lib_fix.so paper_2105_05879_b200/libfst_b200.so
