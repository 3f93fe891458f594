cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e"
timeout 600 $CMD > gpurun_out/ev_plain.json 2> gpurun_out/ev_plain.err; rc=$?; echo "plain rc=$rc"
if [ $rc -eq 0 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fwht|stream_kernel|draw_kernel|identity_kernel|qtable|qtrans|row_norm" -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
fi
