cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for st in 3 5 7 10; do
  FSTG_STREAM_STAGES=$st timeout 600 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu > gpurun_out/st_$st.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/st_$st.json')); print('stages $st value', round(d['value']), 'frac', round(d['roofline']['frac'],3))"
done
