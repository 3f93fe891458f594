set -u
cd "${GRAFT_REPO_ROOT:-.}"
cp paper_2105_05879_b200/libfst_b200.so /tmp/lib_keep.so
for rep in 1 2 3; do
  echo "== ws:  $(timeout 300 python tools/prof_preprocess.py 4096 2>&1 | tr '\n' ' ' | sed 's/GB [0-9.]* GB.s [0-9.]*//g')"
  echo "== old: $(FSTG_SKETCH_WS=0 timeout 300 python tools/prof_preprocess.py 4096 2>&1 | tr '\n' ' ' | sed 's/GB [0-9.]* GB.s [0-9.]*//g')"
done
for v in nostore nocompute; do
  cp tools/variants/lib_$v.so paper_2105_05879_b200/libfst_b200.so
  echo "== $v:  $(timeout 300 python tools/prof_preprocess.py 4096 2>&1 | tr '\n' ' ' | sed 's/GB [0-9.]* GB.s [0-9.]*//g')"
done
cp /tmp/lib_keep.so paper_2105_05879_b200/libfst_b200.so
