cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in k14nt256 k14nt128; do
cp tools/variants/lib_$v.so paper_2105_05879_b200/libfst_b200.so
timeout 900 python bench.py --config 4 --steps 1 --warmup 1 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "$v c4 rc=$?"; tail -2 gpurun_out/bench_c4.err
python -c "
import json; d=json.load(open('gpurun_out/bench_c4.json')); print(round(d['value']), d['preprocess']['kerdock_pass_ms'], d['ms_per_step'])"
done
