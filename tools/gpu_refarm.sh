cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
start=$(date +%s); timeout 900 python bench.py --impl reference > gpurun_out/ref_arm.json 2> gpurun_out/ref_arm.err; echo "ref rc=$? secs=$(( $(date +%s) - start ))"; tail -2 gpurun_out/ref_arm.err; cat gpurun_out/ref_arm.json
