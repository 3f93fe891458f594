cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
ARGS2="--steps 1 --warmup 1 --no-e2e --no-cpu --batch 4096"
timeout 600 python bench.py $ARGS2 > gpurun_out/plain2.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 1 -c 1 -o gpurun_out/prof_stream3 python bench.py $ARGS2 > gpurun_out/ncu_stream.log 2>&1; echo "stream full rc=$?"
