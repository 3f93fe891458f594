cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_default.err
python - <<'PY'
import json; d=json.load(open('gpurun_out/bench_default.json'))
print('value', round(d['value']), 'e2e', round(d['e2e']['value']), 'frac', round(d['roofline']['frac'],3), 'pre', round(d['preprocess']['ms'],1), 'clk', d['clocks'])
print(json.dumps(d['cpu_baseline'], indent=1))
PY
