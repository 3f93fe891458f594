# tests + bench + preprocess timing in one call
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/gpu_tests.log
timeout 300 python tools/prof_preprocess.py 256 > gpurun_out/prof_pre_plain.log 2>&1; cat gpurun_out/prof_pre_plain.log
timeout 900 python bench.py "$@" > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print('value', d['value'], 'frac', d['roofline']['frac'], 'pre_ms', d['preprocess']['ms'], 'pre_frac', d['preprocess']['roofline']['frac'], 'e2e', (d['e2e'] or {}).get('value'), 'cpu', (d['cpu_baseline'] or {}).get('value'), 'support', d['config']['mean_support'])"
