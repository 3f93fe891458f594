cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for dbg in 0 1 2; do
  FSTG_STREAM_DEBUG=$dbg timeout 600 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu > gpurun_out/dbg_$dbg.json 2>gpurun_out/dbg_$dbg.err
  python -c "import json; d=json.load(open('gpurun_out/dbg_$dbg.json')); print('debug $dbg value', d['value'], 'frac', d['roofline']['frac'])"
done
