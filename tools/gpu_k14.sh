# k = 14 retain-sampled Kerdock pass: timings at full / per-basis request load, retain tests, optional ncu capture
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv,noheader
if [ "${K14_TESTS:-1}" = 1 ]; then
timeout 900 python -m pytest tests/test_gpu_retain.py -x -q --timeout 600 -m gpu > gpurun_out/retain_tests.log 2>&1; echo "retain tests rc=$?"; tail -1 gpurun_out/retain_tests.log; grep -E "^E " gpurun_out/retain_tests.log | head -5
fi
for req in 6144000 0; do timeout 300 python tools/prof_k14.py 1024 $req 2>&1 | tail -1; done
if [ "${K14_NCU:-0}" = 1 ]; then
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:fwht_tmem_kernel --launch-count 1 -o gpurun_out/k14_full -f python tools/prof_k14.py 256 6144000 > gpurun_out/ncu_k14.log 2>&1; echo "ncu rc=$?"; tail -1 gpurun_out/ncu_k14.log
fi
