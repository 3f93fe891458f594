# configs 1 / 2 stream A/B of tools/variants/lib_*.so (same box, alternated)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
cp paper_2105_05879_b200/libfst_b200.so /tmp/lib_keep.so
for rep in 1 2; do for v in ${VARIANTS:-base}; do
  cp tools/variants/lib_$v.so paper_2105_05879_b200/libfst_b200.so
  for c in ${CONFIGS:-2 1}; do
    timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/cv.json 2>gpurun_out/cv.err
    python -c "
import json; d=json.load(open('gpurun_out/cv.json')); print('$v config $c', round(d['value']), d['clocks']['sm_mhz'])" || tail -2 gpurun_out/cv.err
  done
done; done
cp /tmp/lib_keep.so paper_2105_05879_b200/libfst_b200.so
