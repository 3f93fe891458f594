cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_retain.py -x -q --timeout 600 -k "preprocess or retain or sample or config4 or gathered" > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 300 python tools/prof_preprocess.py 4096 2>&1 | tail -1
timeout 900 python bench.py --config 4 --steps 1 --warmup 1 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "c4 rc=$?"; tail -2 gpurun_out/bench_c4.err
python -c "
import json; d=json.load(open('gpurun_out/bench_c4.json')); print('c4', round(d['value']), d['preprocess'])"
