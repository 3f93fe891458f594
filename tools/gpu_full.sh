cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q --timeout 900 -m gpu > gpurun_out/gpu_all.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gpu_all.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_full.err
python - <<'PY'
import json; d=json.load(open('gpurun_out/bench_full.json'))
print('value', round(d['value']), 'e2e', round(d['e2e']['value']), 'frac', round(d['roofline']['frac'],3), 'pre', round(d['preprocess']['ms'],1), 'cpu', d.get('cpu_baseline',{}).get('value'), 'clk', d['clocks'])
PY
