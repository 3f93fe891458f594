# config-4 step vs row-block size (pool retained), same box
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do for rb in ${RBS:-0 3072 2048 1536}; do
  timeout 900 python bench.py --config 4 --steps 2 --warmup 1 --row-block $rb > gpurun_out/c4rb.json 2> gpurun_out/c4rb.err
  python -c "
import json; d=json.load(open('gpurun_out/c4rb.json')); print('row_block $rb', round(d['value']), round(d['ms_per_step']), round(d['preprocess']['kerdock_pass_ms']), d['preprocess']['step_breakdown_ms'])" || tail -2 gpurun_out/c4rb.err
done; done
