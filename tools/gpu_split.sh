cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q --timeout 900 -m gpu > gpurun_out/split_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/split_tests.log; grep -E "^E |FAILED" gpurun_out/split_tests.log | head -5
run() { timeout 300 env $4 python bench.py --config $1 --steps $2 --warmup 3 --no-cpu > gpurun_out/rg.json 2>gpurun_out/rg.err; python -c "
import json,sys; d=json.load(open('gpurun_out/rg.json')); print(sys.argv[1], round(d['value']), 'e2e', d['e2e'] and round(d['e2e']['value']), d['clocks']['sm_mhz'])" "$3 config $1" 2>/dev/null || echo "$3 config $1 FAILED"; }
run 1 10 split; run 1 10 nosplit FSTG_NO_BATCH_SPLIT=1; run 3 3 split
