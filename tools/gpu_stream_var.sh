cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
run() { timeout 300 env "$@" python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bv.json 2>gpurun_out/bv.err; python -c "
import json,sys; d=json.load(open('gpurun_out/bv.json')); print(sys.argv[1], round(d['value']), 'frac', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" "$*"; grep l2persist gpurun_out/bv.err | head -1; }
for x in 0 1 0 1; do run FSTG_STREAM_L2PERSIST=$x; done
