set -u
cd "${GRAFT_REPO_ROOT:-.}"
FSTG_SKETCH_BPC=32 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_production.py -x -q --timeout 600 -m gpu -k "sketch or preprocess or k12" > gpurun_out/pre_tests.log 2>&1
echo "tests rc=$?"; tail -1 gpurun_out/pre_tests.log
run() { echo "== $1: $(env $2 timeout 300 python tools/prof_preprocess.py 4096 2>&1 | tr '\n' ' ' | sed 's/GB [0-9.]* GB.s [0-9.]*//g; s/preprocess_ms//g')"; }
for rep in 1 2 3; do
  for b in 24 32 48 64; do
    run "cl1 bpc$b" "FSTG_SKETCH_CL=1 FSTG_SKETCH_BPC=$b"
  done
  run "cl2 bpc32" "FSTG_SKETCH_CL=2 FSTG_SKETCH_BPC=32"
  run "cl2 bpc64" "FSTG_SKETCH_CL=2 FSTG_SKETCH_BPC=64"
  run "old      " "FSTG_SKETCH_WS=0"
done
