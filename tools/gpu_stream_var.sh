cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
run() { timeout 300 env $3 python bench.py --config $2 --steps $4 --warmup 3 --no-cpu --no-e2e > gpurun_out/bv.json 2>gpurun_out/bv.err; python -c "
import json,sys; d=json.load(open('gpurun_out/bv.json')); print(sys.argv[1], round(d['value']), d['clocks']['sm_mhz'])" "$1 config $2"; }
for lib in old new old new; do cp tools/variants/lib_$lib.so paper_2105_05879_b200/libfst_b200.so; run $lib 3 X=1 3; done
cp tools/variants/lib_new.so paper_2105_05879_b200/libfst_b200.so; run new 1 X=1 10; run new 2 X=1 10
timeout 1500 python -m pytest tests -x -q --timeout 900 -m gpu > gpurun_out/split_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/split_tests.log
