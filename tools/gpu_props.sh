cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_properties.py -x -q --timeout 600 -m gpu > gpurun_out/props.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/props.log; grep -E "^E " gpurun_out/props.log | head -10
