cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_retain.py -x -q --timeout 600 -m gpu > gpurun_out/design_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/design_tests.log; grep -E "^E |Error" gpurun_out/design_tests.log | head -10
