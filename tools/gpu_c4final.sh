cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q --timeout 900 -m gpu > gpurun_out/final_tests.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/final_tests.log; grep -E "^FAILED" gpurun_out/final_tests.log | head
timeout 900 python bench.py --config 4 --steps 2 --warmup 1 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "c4 rc=$?"; tail -2 gpurun_out/bench_c4.err
python -c "
import json; d=json.load(open('gpurun_out/bench_c4.json')); print(round(d['value']), d['preprocess']['kerdock_pass_ms'], d['ms_per_step'], d['preprocess']['roofline']['frac'], d['clocks'])"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:fwht_tmem_kernel --launch-count 1 -o gpurun_out/k14_final -f python tools/prof_k14.py 256 6144000 > gpurun_out/ncu_k14.log 2>&1; echo "ncu rc=$?"
