cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_verifiers.py -x -q -s --timeout 600 -m gpu > gpurun_out/verify_tests.log 2>&1; echo "pytest rc=$?"; grep -E "k=|passed|failed|Error|assert" gpurun_out/verify_tests.log | tail -20
