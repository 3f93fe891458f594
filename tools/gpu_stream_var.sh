cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
run() { timeout 300 env "$@" python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bv.json 2>/dev/null; python -c "
import json,sys; d=json.load(open('gpurun_out/bv.json')); print(sys.argv[1], round(d['value']), 'frac', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" "$*"; }
for r in 6 4 3; do
  cp tools/variants/lib_r$r.so paper_2105_05879_b200/libfst_b200.so
  echo "rstages $r"
  run FSTG_STREAM_XBUFS=2
  run FSTG_STREAM_XBUFS=2 FSTG_STREAM_STAGES=6
done
cp tools/variants/lib_r6.so paper_2105_05879_b200/libfst_b200.so
