cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CMD="python tools/prof_preprocess.py 1024"
timeout 300 $CMD > gpurun_out/fwht_plain.log 2>&1; rc=$?; echo "plain rc=$rc"; tail -1 gpurun_out/fwht_plain.log
if [ $rc -eq 0 ]; then
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:fwht_tmem_kernel --launch-count 1 -o gpurun_out/fwht_full -f $CMD > gpurun_out/ncu_fwht.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_fwht.log
fi
