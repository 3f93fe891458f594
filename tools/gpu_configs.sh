cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_experiment.py -m gpu -x -q --timeout 300 > gpurun_out/exp_tests.log 2>&1; echo "exp tests rc=$?"; tail -2 gpurun_out/exp_tests.log
for c in 1 2; do timeout 600 python bench.py --config $c --steps 5 --warmup 2 > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo "config $c rc=$?"; tail -2 gpurun_out/bench_c$c.err; done
timeout 900 python bench.py --config 5 --steps 4 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "config 5 rc=$?"; tail -2 gpurun_out/bench_c5.err
