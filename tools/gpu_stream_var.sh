cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
run() { timeout 300 env "$@" python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bv.json 2>gpurun_out/bv.err; python -c "
import json,sys; d=json.load(open('gpurun_out/bv.json')); print(sys.argv[1], round(d['value']), 'frac', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" "$*"; }
for c in cb0 cb1 cb0 cb1; do
  cp tools/variants/lib_$c.so paper_2105_05879_b200/libfst_b200.so
  echo "$c"; run FSTG_STREAM_DEBUG=0
done
cp tools/variants/lib_cb1.so paper_2105_05879_b200/libfst_b200.so
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -m gpu > gpurun_out/stream_tests.log 2>&1; echo "pytest(cb1) rc=$?"; tail -2 gpurun_out/stream_tests.log
cp tools/variants/lib_cb0.so paper_2105_05879_b200/libfst_b200.so
