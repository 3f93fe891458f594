cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
for c in 1 2; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_config$c.json 2> gpurun_out/bench_config$c.err; echo "config $c rc=$?"; done
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 > gpurun_out/bench_config5.json 2> gpurun_out/bench_config5.err; echo "config 5 rc=$?"
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench_full.json')); print('c3', round(d['value']), 'e2e', round(d['e2e']['value']), 'frac', round(d['roofline']['frac'],3), 'pre', round(d['preprocess']['ms'],1), 'cpu', round(d['cpu_baseline']['value']), d['cpu_baseline'].get('paper_convention',{}).get('value'), d['clocks'])
for c in (1,2):
    d=json.load(open(f'gpurun_out/bench_config{c}.json')); print('c%d'%c, round(d['value']), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'])
d=json.loads(open('gpurun_out/bench_config5.json').readline())
print([(r['s'], r['eps'], round(r['stream_vectors_per_s'])) for r in d['sweep']])
PY
