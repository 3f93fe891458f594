cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
# functional test only (2 ranks share cuda:0 over gloo): checks the N>1 host path runs to completion
FSTG_BENCH_ONE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --config 2 --steps 2 --warmup 1 --no-cpu > gpurun_out/mr.json 2> gpurun_out/mr.err; echo "torchrun rc=$?"; tail -5 gpurun_out/mr.err; cat gpurun_out/mr.json | cut -c1-600
FSTG_BENCH_ONE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err; echo "ref torchrun rc=$?"; tail -3 gpurun_out/mr_ref.err; wc -l gpurun_out/mr_ref.json
