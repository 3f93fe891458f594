cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
free -g | head -2
timeout 900 python bench.py "$@" > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -3 gpurun_out/bench.err
cat gpurun_out/bench.json
