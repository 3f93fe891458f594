cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in 0 1 0 1; do
  cp tools/variants/lib_tma$c.so paper_2105_05879_b200/libfst_b200.so
  echo -n "tma $c: "; timeout 300 python tools/prof_preprocess.py 4096 2>&1 | tail -1
done
cp tools/variants/lib_tma1.so paper_2105_05879_b200/libfst_b200.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_retain.py tests/test_gpu_properties.py tests/test_persist.py -x -q --timeout 600 -m gpu > gpurun_out/tma_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/tma_tests.log; grep -E "^E " gpurun_out/tma_tests.log | head -5
