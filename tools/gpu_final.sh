cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q --timeout 900 -m gpu > gpurun_out/final_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/final_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/ref_final.json 2> gpurun_out/ref_final.err; echo "ref rc=$?"
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench_final.json'))
print('value', round(d['value']), 'e2e', round(d['e2e']['value']), 'frac', round(d['roofline']['frac'],3), 'pre', round(d['preprocess']['ms'],1), 'launches', d['gpu_launches'], 'clk', d['clocks'])
print('cpu', json.dumps({k: (v if not isinstance(v, dict) else {kk: vv for kk, vv in v.items() if kk in ('value','extrapolated_s')}) for k, v in d['cpu_baseline'].items() if k in ('value','single_core','paper_convention')}))
r=json.load(open('gpurun_out/ref_final.json')); print('reference arm', round(r['value']), r['impl'])
PY
