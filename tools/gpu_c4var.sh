# config-4 step A/B of tools/variants/lib_*.so (same box, alternated)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
cp paper_2105_05879_b200/libfst_b200.so /tmp/lib_keep.so
for rep in 1 2; do for v in ${VARIANTS:-base}; do
  cp tools/variants/lib_$v.so paper_2105_05879_b200/libfst_b200.so
  timeout 900 python bench.py --config 4 --steps 2 --warmup 1 > gpurun_out/c4v.json 2> gpurun_out/c4v.err
  python -c "
import json; d=json.load(open('gpurun_out/c4v.json')); print('$v', round(d['value']), round(d['ms_per_step']), round(d['preprocess']['kerdock_pass_ms']), d['preprocess']['step_breakdown_ms']['stream_tail'], d['preprocess']['step_breakdown_ms']['stream_partial'])" || tail -2 gpurun_out/c4v.err
done; done
cp /tmp/lib_keep.so paper_2105_05879_b200/libfst_b200.so
