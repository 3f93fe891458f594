# GPU tests + headline bench (no CPU baseline) + config 5 sweep summary
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 900 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -2 gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print('value', round(d['value']), 'frac', round(d['roofline']['frac'],3), 'pre_ms', round(d['preprocess']['ms'],1), 'e2e', round(d['e2e']['value']), 'support', d['config']['mean_support'], d['clocks'])"
if [ "$1" = "sweep" ]; then
timeout 900 python bench.py --config 5 --steps 4 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "config 5 rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_c5.json'))
for r in d['sweep']: print(r['s'], r['eps'], 'stream', round(r['stream_vectors_per_s']), 'frac', round(r['stream_roofline_frac'],3), 'sgemm', round(r['dense_sgemm_vectors_per_s']), 'match', r['support_match_vs_exact'])"
fi
