cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_retain.py -x -q --timeout 600 -m gpu > gpurun_out/stream_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/stream_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_s.json 2> gpurun_out/bench_s.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_s.err
python - <<'PY'
import json; d=json.load(open('gpurun_out/bench_s.json'))
print('value', round(d['value']), 'e2e', round(d['e2e']['value']), 'frac', round(d['roofline']['frac'],3), 'clk', d['clocks'])
PY
