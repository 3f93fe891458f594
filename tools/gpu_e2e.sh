cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py tests/test_persist.py -x -q --timeout 600 -m gpu > gpurun_out/e2e_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/e2e_tests.log
for c in 1 2 3; do
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err; echo "bench $c rc=$?"
python - <<'PY'
import json; d=json.load(open('gpurun_out/bench_e2e.json'))
print('value', round(d['value']), 'e2e', round(d['e2e']['value']), 'ratio', round(d['e2e']['value']/d['value'],3), d['clocks']['sm_mhz'])
PY
done
