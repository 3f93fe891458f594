cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in 1 2 4 1 4; do
  cp tools/variants/lib_cl$c.so paper_2105_05879_b200/libfst_b200.so
  echo -n "cluster $c: "; timeout 300 python tools/prof_preprocess.py 4096 2>&1 | tail -1
done
for c in 2 4; do
  cp tools/variants/lib_cl$c.so paper_2105_05879_b200/libfst_b200.so
  timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -m gpu -k "preprocess or config3" > gpurun_out/cl_tests.log 2>&1; echo "cluster $c pytest rc=$?"; tail -1 gpurun_out/cl_tests.log
done
cp tools/variants/lib_cl1.so paper_2105_05879_b200/libfst_b200.so
