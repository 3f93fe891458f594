cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
run() { timeout 300 python bench.py --config $2 --steps $3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bv.json 2>gpurun_out/bv.err; python -c "
import json,sys; d=json.load(open('gpurun_out/bv.json')); print(sys.argv[1], round(d['value']), d['clocks']['sm_mhz'])" "$1 config $2"; }
for lib in old new old new old new; do cp tools/variants/lib_$lib.so paper_2105_05879_b200/libfst_b200.so; run $lib 3 3; done
cp tools/variants/lib_new.so paper_2105_05879_b200/libfst_b200.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_retain.py -x -q --timeout 600 -m gpu 2>&1 | tail -1
