#!/usr/bin/env bash
# One entry point for every GPU-box measurement (run through gpurun):
#   /usr/local/graft/bin/gpurun --timeout S -- 'bash tools/gpu.sh <task> [args]'
# Outputs land in gpurun_out/; summaries worth keeping are copied into profiles/.
#
# tasks
#   tests [pytest args]        GPU test suite (default: all -m gpu tests)
#   final                      round-end check: GPU tests, smoke(), headline bench, reference arm
#   bench [bench.py args]      one bench.py run -> gpurun_out/bench.json
#   records                    configs 1 / 2 / 3 / 5 (+ config 1 choose_params) -> gpurun_out/bench_*.json
#   config4 [bench args]       retain tests + bench.py --config 4
#   launches                   ncu launch list (gpu__time_duration) of a short config-3 bench
#   ncu stream|fwht|k14        ncu --set full capture of the top kernel -> gpurun_out/<what>_full.ncu-rep
#   k14 [rows] [requests]      k = 14 retain pass timings (tools/prof_k14.py)
#   ab <lib_a> <lib_b> -- cmd  alternate two library builds (tools/variants/lib_*.so) under one command
#   multirank [config]         N > 1 host path on one GPU (2 ranks over gloo; functional, not a measurement)
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
task=${1:-final}
shift || true

summ() {  # one-line summary of a bench JSON line
  python - "$1" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
keys = {k: d.get(k) for k in ("value", "ms_per_step", "n_gpus")}
if d.get("e2e"):
    keys["e2e"] = round(d["e2e"]["value"])
if "roofline" in d:
    keys["frac"] = round(d["roofline"]["frac"], 3)
if d.get("parity"):
    keys["parity"] = d["parity"]["status"]
if "preprocess" in d:
    keys["pre_ms"] = d["preprocess"].get("ms") or d["preprocess"].get("kerdock_pass_ms")
keys["clocks"] = d.get("clocks")
print(json.dumps(keys))
PY
}

case "$task" in
  tests)
    timeout 2400 python -m pytest tests -q --timeout 900 -m gpu "$@" > gpurun_out/gpu_tests.log 2>&1
    echo "pytest rc=$?"; tail -3 gpurun_out/gpu_tests.log; grep -E "^E " gpurun_out/gpu_tests.log | head -5 ;;
  final)
    timeout 2400 python -m pytest tests -q --timeout 900 -m gpu > gpurun_out/final_tests.log 2>&1
    echo "pytest rc=$?"; tail -2 gpurun_out/final_tests.log
    timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
    timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
    summ gpurun_out/bench_final.json
    timeout 900 python bench.py --impl reference > gpurun_out/ref_final.json 2> gpurun_out/ref_final.err; echo "ref rc=$?"
    summ gpurun_out/ref_final.json ;;
  bench)
    timeout 1800 python bench.py "$@" > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
    tail -3 gpurun_out/bench.err; summ gpurun_out/bench.json ;;
  records)
    timeout 900 python bench.py > gpurun_out/bench_config3.json 2> gpurun_out/bench_config3.err; echo "config 3 rc=$?"
    for c in 1 2; do
      timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_config$c.json 2> gpurun_out/bench_config$c.err
      echo "config $c rc=$?"
    done
    timeout 900 python bench.py --config 1 --choose-params --steps 5 --warmup 3 > gpurun_out/bench_config1_cp.json \
      2> gpurun_out/bench_config1_cp.err; echo "config 1 choose_params rc=$?"
    timeout 1800 python bench.py --config 5 --steps 4 --warmup 3 > gpurun_out/bench_config5.json 2> gpurun_out/bench_config5.err
    echo "config 5 rc=$?"
    for f in config3 config1 config2 config1_cp; do echo -n "$f "; summ gpurun_out/bench_$f.json; done ;;
  config4)
    timeout 900 python -m pytest tests/test_gpu_retain.py -x -q --timeout 600 -m gpu > gpurun_out/retain_tests.log 2>&1
    echo "retain tests rc=$?"; tail -1 gpurun_out/retain_tests.log
    timeout 1800 python bench.py --config 4 --steps 2 --warmup 1 "$@" > gpurun_out/bench_config4.json 2> gpurun_out/bench_config4.err
    echo "config 4 rc=$?"; summ gpurun_out/bench_config4.json ;;
  launches)
    CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity"
    timeout 600 $CMD > gpurun_out/launch_plain.json 2> gpurun_out/launch_plain.err; rc=$?; echo "plain rc=$rc"
    if [ $rc -eq 0 ]; then
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
        -k regex:"fwht|stream_kernel|draw_kernel|identity_kernel|qtable|qtrans|row_norm|narrow" \
        --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
    fi ;;
  ncu)
    what=${1:-stream}
    case "$what" in
      stream) CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-parity"; K="-k regex:stream_kernel --launch-skip 3 --launch-count 1" ;;
      fwht)   CMD="python tools/prof_preprocess.py 1024"; K="-k regex:fwht --launch-count 1" ;;
      k14)    CMD="python tools/prof_k14.py 256 6144000"; K="-k regex:fwht14 --launch-count 1" ;;
      *) echo "unknown ncu target $what"; exit 2 ;;
    esac
    timeout 600 $CMD > gpurun_out/ncu_plain.log 2>&1; rc=$?; echo "plain rc=$rc"
    if [ $rc -eq 0 ]; then
      timeout 1800 ncu --set full --clock-control none --import-source on $K -o gpurun_out/${what}_full -f $CMD \
        > gpurun_out/ncu_$what.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_$what.log
    fi ;;
  k14)
    rows=${1:-1024}; req=${2:-6144000}
    for r in $req 0; do timeout 300 python tools/prof_k14.py $rows $r 2>&1 | tail -1; done ;;
  ab)
    a=$1; b=$2; shift 3
    cp paper_2105_05879_b200/libfst_b200.so /tmp/lib_keep.so
    for v in $a $b $a $b; do
      cp tools/variants/lib_$v.so paper_2105_05879_b200/libfst_b200.so
      echo "== $v: $(timeout 900 "$@" 2>&1 | tail -1)"
    done
    cp /tmp/lib_keep.so paper_2105_05879_b200/libfst_b200.so ;;
  multirank)
    c=${1:-2}
    FSTG_BENCH_ONE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
      --master-addr 127.0.0.1 --master-port 29533 bench.py --config $c --steps 2 --warmup 1 --no-cpu \
      > gpurun_out/multirank.json 2> gpurun_out/multirank.err; echo "torchrun rc=$?"; tail -3 gpurun_out/multirank.err ;;
  *)
    echo "unknown task $task"; exit 2 ;;
esac
