cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_properties.py tests/test_cpp_api.py -x -q --timeout 600 -m gpu > gpurun_out/helpers.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/helpers.log; grep -E "^E " gpurun_out/helpers.log | head -8
