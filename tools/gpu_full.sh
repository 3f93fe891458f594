# full evidence run: tests, smoke, bench (with CPU baseline), ncu launch list, ncu full captures
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -2 gpurun_out/bench.err
ARGS="--steps 2 --warmup 1 --no-e2e --no-cpu --batch 16384"
timeout 600 python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 300 python tools/prof_preprocess.py 256 > gpurun_out/prof_pre_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwht12 -s 0 -c 1 -o gpurun_out/prof_fwht python tools/prof_preprocess.py 256 > gpurun_out/ncu_fwht.log 2>&1; echo "fwht full rc=$?"
ARGS2="--steps 1 --warmup 1 --no-e2e --no-cpu --batch 4096"
timeout 600 python bench.py $ARGS2 > gpurun_out/plain2.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 1 -c 1 -o gpurun_out/prof_stream python bench.py $ARGS2 > gpurun_out/ncu_stream.log 2>&1; echo "stream full rc=$?"
