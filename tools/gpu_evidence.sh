cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e"
timeout 600 $CMD > gpurun_out/ev_plain.json 2> gpurun_out/ev_plain.err; rc=$?; echo "plain rc=$rc"
if [ $rc -eq 0 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_kernel --launch-skip 1 --launch-count 1 -o gpurun_out/stream_full2 -f $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
fi
for c in 1 2; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_config$c.json 2> gpurun_out/bench_config$c.err; echo "config $c rc=$?"; done
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 > gpurun_out/bench_config5.json 2> gpurun_out/bench_config5.err; echo "config 5 rc=$?"
ls -la gpurun_out/*.ncu-rep gpurun_out/launches.csv
