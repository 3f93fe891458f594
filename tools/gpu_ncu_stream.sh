cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e"
timeout 300 $CMD > gpurun_out/ncu_pre.json 2> gpurun_out/ncu_pre.err; rc=$?; echo "plain rc=$rc"
if [ $rc -eq 0 ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_kernel --launch-skip 3 --launch-count 1 \
    -o gpurun_out/stream_full -f $CMD > gpurun_out/ncu_run.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_run.log
fi
ls -la gpurun_out/stream_full.ncu-rep
