set -u
cd "${GRAFT_REPO_ROOT:-.}"
cp paper_2105_05879_b200/libfst_b200.so /tmp/lib_keep.so
run() { echo "== $1: $(env $2 timeout 300 python tools/prof_preprocess.py 4096 2>&1 | tr '\n' ' ' | sed 's/GB [0-9.]* GB.s [0-9.]*//g; s/preprocess_ms//g')"; }
cp tools/variants/lib_lag1.so paper_2105_05879_b200/libfst_b200.so
FSTG_SKETCH_CL=4 timeout 900 python -m pytest tests/test_gpu_production.py -x -q --timeout 600 -m gpu -k "k12" 2>&1 | tail -1
for rep in 1 2 3; do
  cp tools/variants/lib_lag1.so paper_2105_05879_b200/libfst_b200.so
  run "lag1 cl2 bpc64 " "FSTG_SKETCH_CL=2 FSTG_SKETCH_BPC=64"
  run "lag1 cl2 bpc128" "FSTG_SKETCH_CL=2 FSTG_SKETCH_BPC=128"
  run "lag1 cl4 bpc64 " "FSTG_SKETCH_CL=4 FSTG_SKETCH_BPC=64"
  run "lag1 cl4 bpc128" "FSTG_SKETCH_CL=4 FSTG_SKETCH_BPC=128"
  cp /tmp/lib_keep.so paper_2105_05879_b200/libfst_b200.so
  run "lag0 cl2 bpc64 " "FSTG_SKETCH_CL=2 FSTG_SKETCH_BPC=64"
  run "lag0 cl4 bpc64 " "FSTG_SKETCH_CL=4 FSTG_SKETCH_BPC=64"
done
