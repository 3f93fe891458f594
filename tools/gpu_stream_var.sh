cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
run() { timeout 300 env "$@" python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bv.json 2>gpurun_out/bv.err; python -c "
import json,sys; d=json.load(open('gpurun_out/bv.json')); print(sys.argv[1], round(d['value']), 'frac', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" "$*"; }
for c in rp0 rp1 rp0 rp1; do
  cp tools/variants/lib_$c.so paper_2105_05879_b200/libfst_b200.so
  echo "$c"; run FSTG_STREAM_DEBUG=0
done
cp tools/variants/lib_rp1.so paper_2105_05879_b200/libfst_b200.so
