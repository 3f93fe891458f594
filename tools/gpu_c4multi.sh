cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_retain.py tests/test_cpp_api.py -x -q --timeout 600 -m gpu > gpurun_out/c4m_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/c4m_tests.log
timeout 900 python bench.py --config 4 --steps 1 --warmup 1 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "c4 rc=$?"; tail -2 gpurun_out/bench_c4.err
cat gpurun_out/bench_c4.json
