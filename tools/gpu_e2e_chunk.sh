# e2e (host buffers) vs first-chunk size, config 2 (4096 vectors/step) and config 1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do for fc in default 512 1024 2048; do
  if [ $fc = default ]; then unset FSTG_FIRST_CHUNK; else export FSTG_FIRST_CHUNK=$fc; fi
  timeout 300 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu > gpurun_out/ce.json 2>gpurun_out/ce.err
  python -c "
import json; d=json.load(open('gpurun_out/ce.json')); print('first_chunk $fc config 2 value', round(d['value']), 'e2e', round(d['e2e']['value']))" || tail -2 gpurun_out/ce.err
done; done
