# config-4 step experiments (same box): env / row-block settings, per-scope breakdown
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
run() {
  env $2 timeout 900 python bench.py --config 4 --steps 2 --warmup 1 $3 > gpurun_out/c4x.json 2> gpurun_out/c4x.err
  python -c "
import json,sys; d=json.load(open('gpurun_out/c4x.json')); print('$1', round(d['value']), round(d['ms_per_step']), round(d['preprocess']['kerdock_pass_ms']), d['preprocess'].get('step_breakdown_ms'), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/c4x.err
}
run default "X=1" ""
run notrim "FSTG_NO_TRIM=1" ""
run cl8 "FSTG_RETAIN_CLUSTER=8" ""
run cl0 "FSTG_RETAIN_CLUSTER=0" ""
run rb2048 "X=1" "--row-block 2048"
run rb1024 "X=1" "--row-block 1024"
