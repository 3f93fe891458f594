cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_retain.py -x -q --timeout 600 -m gpu > gpurun_out/design_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/design_tests.log; grep -E "^E " gpurun_out/design_tests.log | head -5
timeout 900 python bench.py --config 4 --steps 2 --warmup 1 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "c4 rc=$?"; tail -2 gpurun_out/bench_c4.err
python -c "
import json; d=json.load(open('gpurun_out/bench_c4.json')); print(round(d['value']), d['preprocess']['kerdock_pass_ms'], d['ms_per_step'])"
