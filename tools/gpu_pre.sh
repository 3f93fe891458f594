cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --timeout 300 -k "preprocess" > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gpu_tests.log
for st in normal cs; do FSTG_FWHT_STORE=$st timeout 300 python tools/prof_preprocess.py 4096 > gpurun_out/prof_pre_$st.log 2>&1; echo "store $st"; cat gpurun_out/prof_pre_$st.log; done
