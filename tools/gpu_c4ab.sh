# config-4 step A/B: current library vs tools/variants/lib_head.so (same box), with host-side timing breakdown
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
cp paper_2105_05879_b200/libfst_b200.so /tmp/lib_new.so
for v in new head new; do
  if [ $v = head ]; then cp tools/variants/lib_head.so paper_2105_05879_b200/libfst_b200.so; else cp /tmp/lib_new.so paper_2105_05879_b200/libfst_b200.so; fi
  timeout 900 python bench.py --config 4 --steps 2 --warmup 1 > gpurun_out/bench_c4_$v.json 2> gpurun_out/bench_c4_$v.err
  python -c "
import json,sys; d=json.load(open('gpurun_out/bench_c4_$v.json')); print('$v', round(d['value']), round(d['ms_per_step']), round(d['preprocess']['kerdock_pass_ms']), d['preprocess'].get('step_breakdown_ms'))"
done
cp /tmp/lib_new.so paper_2105_05879_b200/libfst_b200.so
