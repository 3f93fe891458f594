set -u
cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_production.py -x -q --timeout 600 -m gpu -k "sketch or preprocess or k12 or config3 or fp32" > gpurun_out/pre_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/pre_tests.log
for rep in 1 2; do
  echo "== ws:  $(timeout 300 python tools/prof_preprocess.py 4096 2>&1 | tail -1)"
  echo "== old: $(FSTG_SKETCH_WS=0 timeout 300 python tools/prof_preprocess.py 4096 2>&1 | tail -1)"
done
