cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
run() { timeout 300 env $4 python bench.py --config $1 --steps $2 --warmup 3 --no-cpu --no-e2e > gpurun_out/bv.json 2>gpurun_out/bv.err; python -c "
import json,sys; d=json.load(open('gpurun_out/bv.json')); print(sys.argv[1], round(d['value']), d['clocks']['sm_mhz'])" "$3 $4 config $1" 2>/dev/null || echo "$3 $4 FAILED"; }
for lib in rb4 rb8; do
  cp tools/variants/lib_$lib.so paper_2105_05879_b200/libfst_b200.so
  run 3 3 $lib FSTG_STREAM_RDIRECT=0; run 3 3 $lib FSTG_STREAM_RDIRECT=1
done
cp tools/variants/lib_rb4.so paper_2105_05879_b200/libfst_b200.so
run 3 3 rb4 FSTG_STREAM_RDIRECT=1; run 3 3 rb4 FSTG_STREAM_RDIRECT=0
