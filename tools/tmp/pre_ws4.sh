set -u
cd "${GRAFT_REPO_ROOT:-.}"
run() { echo "== $1: $(env $2 timeout 300 python tools/prof_preprocess.py 4096 2>&1 | tr '\n' ' ' | sed 's/GB [0-9.]* GB.s [0-9.]*//g; s/preprocess_ms//g')"; }
for rep in 1 2 3; do
  run "cl2 bpc128" "FSTG_SKETCH_CL=2"
  run "cl2 bpc32 " "FSTG_SKETCH_CL=2 FSTG_SKETCH_BPC=32"
  run "cl2 bpc512" "FSTG_SKETCH_CL=2 FSTG_SKETCH_BPC=512"
  run "cl1 bpc32 " "FSTG_SKETCH_CL=1 FSTG_SKETCH_BPC=32"
  run "cl1 bpc16 " "FSTG_SKETCH_CL=1 FSTG_SKETCH_BPC=16"
  run "cl1 bpc512" "FSTG_SKETCH_CL=1 FSTG_SKETCH_BPC=512"
  run "old       " "FSTG_SKETCH_WS=0"
done
