set -u
cd "${GRAFT_REPO_ROOT:-.}"
FSTG_SKETCH_CL=4 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_production.py -x -q --timeout 600 -m gpu -k "sketch or preprocess or k12" > gpurun_out/pre_tests.log 2>&1
echo "tests CL=4 rc=$?"; tail -1 gpurun_out/pre_tests.log
FSTG_SKETCH_CL=2 timeout 900 python -m pytest tests/test_gpu_production.py -x -q --timeout 600 -m gpu -k "k12" > gpurun_out/pre_tests2.log 2>&1
echo "tests CL=2 rc=$?"; tail -1 gpurun_out/pre_tests2.log
for rep in 1 2 3; do
  for cl in 1 2 4; do
    echo "== ws cl=$cl: $(FSTG_SKETCH_CL=$cl timeout 300 python tools/prof_preprocess.py 4096 2>&1 | tr '\n' ' ' | sed 's/GB [0-9.]* GB.s [0-9.]*//g')"
  done
  echo "== old: $(FSTG_SKETCH_WS=0 timeout 300 python tools/prof_preprocess.py 4096 2>&1 | tr '\n' ' ' | sed 's/GB [0-9.]* GB.s [0-9.]*//g')"
done
