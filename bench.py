#!/usr/bin/env python
"""Headline benchmark: thresholded-Ax vectors/s at n=4096, s=32 (BASELINE config 3).

One step = one pass of the streaming hot path (draw -> sampled-basis
coefficients -> gather-accumulate -> median-of-means -> top-(widen*s) select ->
exact refinement -> eps threshold) over a batch of B synthetic config-3 vectors
per GPU, J=375, K=2, widen=10 (N = 750 samples / vector).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

N > 1 runs under torchrun (one rank per GPU, NCCL): rank 0 builds A and
broadcasts it over NCCL/NVLink, every rank builds its own sketch replica and
streams its own shard of vectors (global vector ids rank*B + i; weak scaling).
The reference arm (--impl reference) times the reference algorithm's CPU
restatement (oracle/, the reference itself does not build here: no Eigen) on
the host cores of rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

J_DEFAULT, K_DEFAULT, WIDEN = 375, 2, 10
N_DIM, S, EPS = 4096, 32, 0.1
A_SEED, X_SEED = 4096, 20251019
METRIC = "thresholded-Ax vectors/sec at n=4096,s=32 (1/2/4/8 B200); preprocess time"
# FP32 adds/s of the CUDA cores, measured on a B200 at the 1965 MHz max clock (tools/micro/fadd_peak.cu:
# 126 adds/clk/SM for FADD and FADD2 alike; profiles/r01_fadd_peak.txt)
FP32_ADD_PEAK_TADD = 36.7


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--batch", type=int, default=65536, help="vectors per GPU per step")
    ap.add_argument("--J", type=int, default=J_DEFAULT)
    ap.add_argument("--K", type=int, default=K_DEFAULT)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--row-block", type=int, default=0,
                    help="config 4: rows per retain-sampled block (0 = as many as ~70%% of free HBM holds)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--choose-params", action="store_true",
                    help="J, K from choose_params(row_norm_max, gamma = eps/2, eta = 0.1, m), the reference CLI's "
                         "default (cli.hpp:164-172, stream.hpp:58-69), instead of the paper's J=375, K=2")
    ap.add_argument("--no-parity", action="store_true", help="skip the post-timing oracle check of the timed batch")
    ap.add_argument("--config", default="3", choices=["1", "2", "3", "4", "5"],
                    help="BASELINE.json configs: 3 = headline (default); 1, 2 = parity-case workloads; "
                         "5 = s x eps sweep with the dense-GEMM crossover")
    ap.add_argument("--replicate", default="recompute", choices=["recompute", "allgather"],
                    help="sketch replica per GPU: local recompute after the A broadcast, or basis-sharded "
                         "preprocessing + NVLink all-gather")
    return ap.parse_args()


# Read-only DRAM ceiling of the stream kernel's access pattern (random 16 KiB columns, several issuing lanes),
# measured on a B200 with tools/micro/rand_read.cu (profiles/r01_tma_issue.txt: 7,104-7,309 GB/s)
RANDOM_READ_CEILING_GBS = 7250.0


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def bytes_per_vector(N, m, n, want, es=4):
    """Algorithmic bytes per vector as SURVEY.md §8(d) counts them: N sampled columns, want rows of A, x."""
    return es * (N * m + want * n + n)


def dram_bytes_per_vector(N, m, n, es=4):
    """DRAM-resident algorithmic bytes per vector: the N sampled sketch columns and x.

    The `want` gathered rows of A are left out: A (64 MiB at n = 4096) stays L2-resident for the whole
    launch (its rows are loaded with an evict_last policy), which is the rule §8(d) itself applies to
    the L2-resident sign tables. The measured DRAM traffic of the kernel (ncu) is reported beside it;
    traffic / algorithmic is the re-read waste (A-row L2 misses, x re-reads)."""
    return es * (N * m + n)


# DRAM bytes of one stream-kernel launch of 65,536 config-3 vectors, ncu --set full
# (dram__bytes_read.sum + dram__bytes_write.sum), profiles/r02_ncu_stream_kernel_final.txt
NCU_STREAM_DRAM_BYTES_65536 = 837.875902e9 + 3.203679e9
NCU_STREAM_SOURCE = ("profiles/r02_ncu_stream_kernel_final.txt (ncu --set full, one 65,536-vector launch, "
                     "scaled per vector)")


def spread_vectors(B, sms=148, extra=8, seed=0):
    """Vector ids covering every position in the persistent kernel's walk (CTA c handles
    c, c + grid, c + 2 grid, ...): the 1st / 2nd / ... / last vector of several CTAs."""
    grid = min(B, sms)
    rounds = (B + grid - 1) // grid
    ids = set()
    for r in sorted({0, 1, 2, rounds // 2, rounds - 2, rounds - 1}):
        if r < 0:
            continue
        for off in (0, grid // 2, grid - 1):
            v = r * grid + off
            if 0 <= v < B:
                ids.add(v)
    ids.update({B - 1})
    rng = np.random.default_rng(seed)
    target = min(B, len(ids) + extra)
    while len(ids) < target:
        ids.add(int(rng.integers(0, B)))
    return sorted(ids)


def torch_float32():
    import torch
    return torch.float32


def parity_check(fst, sk, A, X, seeds, out, J, K, s_val, eps_val, strict, nvec=32):
    """After timing: outputs of the timed batch for >= nvec spread vectors against the oracle's
    draw_and_gather transform (stream.hpp:184-191, 197-268) on the GPU's own gathered columns,
    in fp64, on exactly the inputs the GPU saw. Bars (BASELINE.json north_star): draws bit-exact;
    supports identical except entries within 1e-6 of eps or at the rank-want estimator cut-off;
    values within 1e-5 relative (fp32) / 1e-12 (fp64 STRICT, where supports must be identical)."""
    from oracle import oracle as orc   # checker only, outside the timed region
    B = X.shape[0]
    ids = list(range(B)) if B <= 2 * nvec else spread_vectors(B, extra=max(0, nvec - 18))
    want = fst.candidate_count(s_val, WIDEN, sk.m)
    p = fst.StreamParams(epsilon=eps_val, s=s_val, J=J, K=K, widen=WIDEN)
    a64 = A.double().cpu().numpy()
    counts = out.counts.cpu().numpy()
    sup, vals = out.support.cpu().numpy(), out.values.cpu().numpy()
    seeds_np = np.asarray(seeds, dtype=np.uint64)
    idx = fst.draw_samples(sk, p, seeds=seeds_np[ids])
    draws_ok = exact = allowed = bit_exact = 0
    max_rel = 0.0
    failures = []
    fast = not strict and X.dtype == torch_float32()
    for q, v in enumerate(ids):
        op = orc.StreamParams(epsilon=eps_val, s=s_val, J=J, K=K, widen=WIDEN, seed=int(seeds_np[v]))
        ref_idx = orc.draw_samples(sk.L, op)
        draws_ok += int(np.array_equal(idx[q], ref_idx))
        x = X[v].double().cpu().numpy()
        cols = sk.gather(ref_idx)
        if fast:
            # bit for bit against the CPU restatement of the FAST kernels' own summation orders
            rk = orc.transform_gathered_fast_order(A.cpu().numpy(), X[v].cpu().numpy(), op, ref_idx, cols)
            c = int(counts[v])
            bit_exact += int(sup[v, :c].tolist() == rk.support.tolist()
                             and vals[v, :c].tobytes() == rk.values.tobytes())
        r = orc.transform_gathered(a64, x, op, ref_idx, cols.astype(np.float64))
        g_sup = sup[v, :counts[v]].tolist()
        g_val = vals[v, :counts[v]].astype(np.float64)
        ri = dict(zip(r.support.tolist(), r.values))
        for i, gv in zip(g_sup, g_val):
            if i in ri:
                max_rel = max(max_rel, abs(gv - ri[i]) / max(abs(ri[i]), 1e-300))
        if g_sup == r.support.tolist():
            exact += 1
            continue
        if strict:
            failures.append(v)
            continue
        ax = a64 @ x
        cut = np.sort(np.abs(r.mu))[::-1][want - 1] if want <= sk.m else 0.0
        ok = all(abs(abs(ax[i]) - eps_val) <= 1e-6 or abs(abs(r.mu[i]) - cut) <= 1e-5 * max(1.0, cut)
                 for i in set(g_sup) ^ set(r.support.tolist()))
        allowed += int(ok)
        if not ok:
            failures.append(v)
    tol = 1e-12 if strict else 1e-5
    ok = draws_ok == len(ids) and not failures and max_rel <= tol and (not fast or bit_exact == len(ids))
    return {"status": "ok" if ok else "FAIL", "vectors_checked": len(ids), "vector_ids": ids,
            "draws_bit_exact": draws_ok, "support_identical": exact, "support_diff_allowed": allowed,
            "failures": failures, "max_value_rel_err": max_rel, "value_tol": tol,
            "kernel_order_bit_exact": bit_exact if fast else None,
            "oracle": "oracle.transform_gathered (fp64 restatement of stream.hpp:197-268) on the GPU's gathered "
                      "columns; inputs = the GPU's exact A and x. fp32 FAST: supports and values also bit-exact "
                      "against oracle.transform_gathered_fast_order (the kernels' summation orders restated)"}


# ------------------------------------------------------------- clocks ----
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# -------------------------------------------------------- CPU baseline ----
def pool_size(N, m, budget=1.5e9):
    """Prepared vectors for the CPU leg: their materialised fp64 columns (P x N x m) within ~1.5 GB."""
    return int(max(1, min(32, budget // (N * m * 8))))


def cpu_sample(a64: np.ndarray, X64: np.ndarray, seeds: np.ndarray, J: int, K: int, threads: int,
               target_s: float, predrawn: bool = False, s_val: int = S, eps_val: float = EPS):
    """The reference algorithm on host cores over a pool of prepared vectors.

    kind "reference": the reference's own stream.hpp/sketch.hpp code compiled from its
    sources (oracle/_ref/libfst_ref.so, built by `make -C oracle ref` against the Eigen-API
    shim; it travels with the repo snapshot). kind "port": the oracle restatement, used when
    that library is absent or for the paper's predrawn convention (which the reference's
    transform() has no entry for).
    The fp64 sketch at n=4096 needs 275 GB of host RAM (the box has ~196 GB), so
    the sampled columns are materialised per vector (A s_ell via BLAS, untimed)
    into host DRAM and the timed loop runs the reference transform() — draws,
    Gray-code coefficients, accumulation over the columns read from DRAM,
    median, top-k, refinement — with each thread on its own vectors."""
    from oracle import oracle as orc
    from oracle import refimpl
    m, n = a64.shape
    k = orc.even_log2_ceil(n)
    _, L = orc.design_params(k)
    P = X64.shape[0]
    N = J * K
    gathered = np.empty((P, N, m), dtype=np.float64)
    for v in range(P):
        p = orc.StreamParams(epsilon=eps_val, s=s_val, J=J, K=K, widen=WIDEN, seed=int(seeds[v]))
        idx = orc.draw_samples(L, p)
        S_ = orc.design_columns(k, n, idx)          # (N, n)
        gathered[v] = S_ @ a64.T                    # column ell = A s_ell
    p = orc.StreamParams(epsilon=eps_val, s=s_val, J=J, K=K, widen=WIDEN)
    kind = "reference" if (refimpl.available() and not predrawn) else "port"
    if kind == "reference":
        run = lambda total: refimpl.bench_gathered(a64, X64, p, seeds, gathered, threads, total)  # noqa: E731
    else:
        run = lambda total: orc.bench_gathered(a64, X64, p, seeds, gathered, L, threads, total, predrawn)  # noqa: E731
    _, t_pool = run(P)
    total = max(P, int(P * max(1.0, target_s / max(t_pool, 1e-3))))
    counts, secs = run(total)
    return {"value": total / secs, "seconds": secs, "vectors": total, "pool": P,
            "pool_support_mean": float(np.mean(counts)), "kind": kind}


def cpu_impl_text(kind: str) -> str:
    if kind == "reference":
        return ("the reference's own transform_with_samples() (stream.hpp, compiled from its sources against the "
                "Eigen-API shim, oracle/_ref/libfst_ref.so; its draw_samples timed per vector)")
    return "reference transform() restated in C++ (oracle/)"


# ------------------------------------------------------------ GPU arm ----
WORKLOADS = {
    "3": dict(n=4096, dtype="fp32", s=32, eps=0.1, B=65536, a="haar", a_seed=4096,
              desc="config3: n=m=4096, s=32, eps=0.1, J={J}, K={K}, widen=10 (N={N}, want=320)",
              data="synthetic (seeded config-3 generator: Haar-orthogonal A, y 32-sparse +-1/sqrt(32) + N(0,1e-6), "
                   "x = A^T y / |.|)"),
    "1": dict(n=256, dtype="fp64", s=8, eps=0.1, B=64, a="haar", a_seed=777,
              desc="config1: n=m=256 fp64, s=8, eps=0.1, 64 vectors/step, J={J}, K={K}, widen=10",
              data="synthetic (Haar-orthogonal A, y 8-sparse +-1/sqrt(8), x = A^T y)"),
    "2": dict(n=1024, dtype="fp32", s=16, eps=0.05, B=4096, a="iid", a_seed=1024,
              desc="config2: n=m=1024 fp32, A iid N(0,1/n), s=16, eps=0.05, 4096 vectors/step, J={J}, K={K}",
              data="synthetic (A iid N(0,1/n), y 16-sparse N(0,1), x = A^-1 y / |.|)"),
}


def make_problem(cfg, A64, B, first, dev, targets=None):
    from paper_2105_05879_b200 import generators
    if cfg is WORKLOADS["1"]:
        return generators.config1_problem(B=B, seed=X_SEED, device=dev, a_seed=cfg["a_seed"], A64=A64,
                                          targets=targets)
    if cfg is WORKLOADS["2"]:
        return generators.config2_problem(B=B, seed=X_SEED, device=dev, a_seed=cfg["a_seed"], first=first, A64=A64,
                                          targets=targets)
    return generators.config3_problem(B=B, seed=X_SEED, device=dev, first=first, A64=A64, targets=targets)


def build_matrix(cfg, dev, gaussian_fill=None):
    """A in fp64 on `dev`: the SeededRng Gaussian fill (library or oracle, bit-identical), then QR
    (Haar) or 1/sqrt(n) scaling (iid); both arms call this, so they get the same A bits."""
    from paper_2105_05879_b200 import generators
    n = cfg["n"]
    if cfg["a"] == "haar":
        return generators.haar_orthogonal(n, cfg["a_seed"], dev, gaussian_fill=gaussian_fill)
    return generators.iid_gaussian(n, cfg["a_seed"], dev, gaussian_fill=gaussian_fill)


def batch_size(args, cfg):
    return args.batch if args.config == "3" else cfg["B"]


def workload_config(args, cfg, world):
    """The `config` object both arms print (identical keys and values)."""
    desc = cfg["desc"].format(J=args.J, K=args.K, N=args.J * args.K)
    if args.choose_params:
        desc += " (J, K from choose_params(row_norm_max, eps/2, 0.1, m): the reference CLI default, cli.hpp:164-172)"
    return {"workload": desc, "vectors_per_gpu_per_step": batch_size(args, cfg), "J": args.J, "K": args.K,
            "widen": WIDEN, "parallelism": f"vector-sharded x{world}, sketch replicated per GPU",
            "l2": ("inputs larger than L2 (137.5 GB sketch; 1 GiB of x per step)" if args.config == "3"
                   else "small config: sketch may be L2-resident")}


def run_b200(args):
    import torch
    import torch.distributed as dist
    from paper_2105_05879_b200 import fst, generators, parallel

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # functional check of the N > 1 host path on a one-GPU box (never a measurement):
    # every rank on cuda:0, gloo collectives; no kernel waits on another rank's
    one_dev = os.environ.get("FSTG_BENCH_ONE_DEVICE") == "1"
    if one_dev:
        local = 0
    torch.cuda.set_device(local)
    dev = f"cuda:{local}"
    if world > 1:
        if one_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(dev))
        dist.barrier()
        nccl = ".".join(map(str, torch.cuda.nccl.version())) if not one_dev else "-"
        print(f"[bench] rank {rank}/{world} on {dev}: {dist.get_backend()} process group up "
              f"(NCCL {nccl}), group size {dist.get_world_size()}", file=sys.stderr, flush=True)

    cfg = WORKLOADS[args.config]
    n_dim = cfg["n"]
    es = 8 if cfg["dtype"] == "fp64" else 4
    # ---- A: built on rank 0, broadcast over NCCL ----
    if rank == 0:
        A64 = build_matrix(cfg, dev)
    else:
        A64 = torch.empty((n_dim, n_dim), dtype=torch.float64, device=dev)
    if world > 1:
        parallel.broadcast_matrix(A64, src=0)
    A32 = A64.contiguous() if es == 8 else A64.float().contiguous()

    # ---- sketch replica per GPU (device time) ----
    fst.profile_enable(True)
    fst.profile_reset()
    gather_ms = 0.0
    if args.replicate == "allgather" and world > 1:
        nk = fst.design_params(fst.even_log2_ceil(n_dim))[0] // 2
        first, count = parallel.basis_shards(nk, world)[rank]
        sk = fst.preprocess_shard(A32, first, first + count, True, device=local)
        full = parallel.sketch_tensor(sk)
        dist.barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record()
        parallel.allgather_basis_shards(full, world, rank, nk, sk.d, sk.column_stride)
        g1.record()
        torch.cuda.synchronize()
        gather_ms = g0.elapsed_time(g1)
    else:
        sk = fst.preprocess(A32, device=local)
    fwht_ms, _ = fst.profile_read("preprocess_fwht")
    ident_ms, _ = fst.profile_read("preprocess_identity")
    pre_ms = parallel.max_over_ranks(sk.preprocess_ms + gather_ms, device=dev)
    sketch_bytes = sk.L * sk.m * es

    if args.choose_params:  # the reference CLI's default regime (cli.hpp:164-172)
        args.J, args.K = fst.choose_params(sk.row_norm_max(), cfg["eps"] / 2, 0.1, sk.m)

    # ---- this rank's shard of the vector stream ----
    B = batch_size(args, cfg)
    first, _ = parallel.vector_shard(rank, world, B)
    prob = make_problem(cfg, A64, B, first, dev)
    X = prob.X
    seeds_dev = torch.from_numpy(prob.seeds.view(np.int64)).to(dev)
    s_val, eps_val = cfg["s"], cfg["eps"]
    p = fst.StreamParams(epsilon=eps_val, s=s_val, J=args.J, K=args.K, widen=WIDEN)
    N = args.J * args.K
    want = fst.candidate_count(s_val, WIDEN, n_dim)
    vdt = torch.float64 if es == 8 else torch.float32
    out = fst.BatchResult(torch.zeros(B, dtype=torch.int32, device=dev),
                          torch.zeros((B, want), dtype=torch.int32, device=dev),
                          torch.zeros((B, want), dtype=vdt, device=dev))
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream

    def step():
        fst.transform_batch(sk, X, p, seeds_dev, out=out, stream=sptr)

    w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i in range(args.warmup):
        if i == args.warmup - 1:
            torch.cuda.synchronize()
            w0.record(stream)
        step()
    w1.record(stream)
    torch.cuda.synchronize()
    # The library's per-launch CUDA-event brackets cost ~15 us of device time per call: inside
    # the timed region for long steps (config 3: 150 ms), in a separate profiled pass of the
    # same K steps for sub-20-ms steps (configs 1 / 2), where they would cost 1-13 %.
    profile_in_timed = w0.elapsed_time(w1) >= 20.0  # the last warm-up step
    if not profile_in_timed:
        fst.profile_enable(False)

    # ---- timed region (device resident) ----
    fst.profile_reset()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    launches = fst.launch_count()
    if not profile_in_timed:  # per-launch kernel times from an identical, untimed, profiled pass
        fst.profile_enable(True)
        fst.profile_reset()
        for _ in range(args.steps):
            step()
        torch.cuda.synchronize()
    stream_ms, stream_launches = fst.profile_read("stream")
    draw_ms, draw_launches = fst.profile_read("draw")
    fst.profile_enable(False)
    ms_max = parallel.max_over_ranks(ms, device=dev)
    counts = out.counts.cpu().numpy()
    value = world * B * args.steps / (ms_max / 1e3)

    # ---- roofline of the dominant kernel (the fused stream kernel) ----
    peak, peak_kind = peaks()
    bvec = bytes_per_vector(N, sk.m, sk.n, want, es)         # SURVEY.md §8(d) count (A rows included)
    dvec = dram_bytes_per_vector(N, sk.m, sk.n, es)          # DRAM-resident algorithmic bytes
    per_launch_ms = stream_ms / max(1, stream_launches)
    vec_per_launch = B * args.steps / max(1, stream_launches)
    achieved = dvec * vec_per_launch / (per_launch_ms / 1e3) / 1e9
    achieved_8d = bvec * vec_per_launch / (per_launch_ms / 1e3) / 1e9
    pre_achieved = sketch_bytes / (fwht_ms + ident_ms) / 1e6 if (fwht_ms + ident_ms) > 0 else None

    # DRAM bytes per launch of the stream kernel from the committed ncu --set full capture
    # (dram__bytes_read.sum + dram__bytes_write.sum of one config-3 launch of 65,536 vectors),
    # scaled to this run's vectors per launch
    traffic, traffic_src = None, None
    if args.config == "3":
        traffic = NCU_STREAM_DRAM_BYTES_65536 / 65536 * vec_per_launch
        traffic_src = NCU_STREAM_SOURCE

    # ---- end to end through the public API with host buffers ----
    e2e = None
    if not args.no_e2e:
        Xh = X.cpu().pin_memory()
        seeds_h = torch.from_numpy(prob.seeds.view(np.int64).copy()).pin_memory()
        oh = fst.BatchResult(torch.zeros(B, dtype=torch.int32).pin_memory(),
                             torch.zeros((B, want), dtype=torch.int32).pin_memory(),
                             torch.zeros((B, want), dtype=vdt).pin_memory())
        for _ in range(max(1, args.warmup)):
            fst.transform_batch(sk, Xh, p, seeds_h, out=oh, stream=sptr)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            fst.transform_batch(sk, Xh, p, seeds_h, out=oh, stream=sptr)
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
        e2e = {"value": world * B * args.steps / parallel.max_over_ranks(e2e_s, device=dev), "unit": "vectors/s",
               "h2d_bytes_per_step": int(B * n_dim * es + B * 8),
               "d2h_bytes_per_step": int(B * 4 + B * want * (4 + es))}
        assert np.array_equal(oh.counts.numpy(), counts), "host-buffer path disagrees with device path"

    # ---- parity of the timed batch's outputs against the oracle (after timing) ----
    parity = None
    if not args.no_parity:
        strict = es == 8
        parity = parity_check(fst, sk, prob.A, X, prob.seeds, out, args.J, args.K, s_val, eps_val, strict)
        print(f"[bench] rank {rank}: parity {parity['status']} ({parity['vectors_checked']} vectors of the timed "
              f"batch vs the oracle, support identical {parity['support_identical']}, "
              f"max value rel err {parity['max_value_rel_err']:.2e}, bit-exact vs the kernel-order "
              f"restatement {parity['kernel_order_bit_exact']})", file=sys.stderr, flush=True)

    # ---- CPU baseline (rank 0, N = 1) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and args.config == "3":
        P = pool_size(N, sk.m)
        a64 = prob.A.double().cpu().numpy()          # exactly the A the GPU computes on
        X64 = X[:P].double().cpu().numpy()
        threads = os.cpu_count() or 1
        r = cpu_sample(a64, X64, prob.seeds[:P], args.J, args.K, threads, args.cpu_seconds)
        cpu = {"value": r["value"], "unit": "vectors/s", "cores": threads, "kind": r["kind"],
               "sample": (f"{r['vectors']} config-3 vectors ({r['pool']} distinct, cycled) over {threads} threads, "
                          f"{r['seconds']:.1f} s: {cpu_impl_text(r['kind'])}, fp64, "
                          f"columns A*s_ell pre-materialised in host DRAM because the 275 GB fp64 sketch "
                          f"exceeds host RAM")}
        # single-core transform, and the reference preprocessing on the
        # host (all threads / 1 thread) on a bounded sample of bases, extrapolated to all 2048
        r1 = cpu_sample(a64, X64, prob.seeds[:P], args.J, args.K, 1, min(3.0, args.cpu_seconds / 3))
        cpu["single_core"] = {"value": r1["value"], "unit": "vectors/s", "cores": 1, "kind": r1["kind"],
                              "sample": f"{r1['vectors']} vectors, {r1['seconds']:.1f} s"}
        rp = cpu_sample(a64, X64, prob.seeds[:P], args.J, args.K, threads, min(4.0, args.cpu_seconds / 3),
                        predrawn=True)
        cpu["paper_convention"] = {"value": rp["value"], "unit": "vectors/s", "cores": threads, "kind": rp["kind"],
                                   "sample": f"{rp['vectors']} vectors, {rp['seconds']:.1f} s; index draws and "
                                             "column gathers outside the clock (experiment.hpp:178-181)"}
        from oracle import oracle as orc
        nk = 2048
        pre_all = orc.bench_preprocess(a64, threads, threads)
        pre_one = orc.bench_preprocess(a64, 1, 1)
        cpu["preprocess"] = {
            "unit": "s", "dtype": "f64",
            "all_threads": {"cores": threads, "sample_bases": threads, "sample_s": pre_all,
                            "extrapolated_s": pre_all * nk / threads},
            "one_thread": {"cores": 1, "sample_bases": 1, "sample_s": pre_one, "extrapolated_s": pre_one * nk},
            "note": ("reference per-basis preprocessing (kerdock_matrix + masked FWHT + transposed stores, "
                     "sketch.hpp:171-196) timed on the first bases and scaled to 2048 Kerdock bases; the full "
                     "275 GB fp64 sketch does not fit host RAM")}

    line = {
        "metric": METRIC if args.config == "3" else f"thresholded-Ax vectors/sec ({cfg['desc'].split(':')[0]})",
        "value": value,
        "unit": "vectors/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_max / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": cfg["dtype"],
        "data": cfg["data"],
        "config": workload_config(args, cfg, world),
        "mean_support": float(np.mean(counts)),
        "preprocess": {"ms": pre_ms, "fwht_ms": fwht_ms, "identity_ms": ident_ms, "allgather_ms": gather_ms,
                       "replicate": args.replicate,
                       "sketch_bytes": sketch_bytes,
                       "roofline": {"bound": "hbm", "achieved": pre_achieved, "peak": peak, "unit": "GB/s",
                                    "frac": (pre_achieved / peak) if pre_achieved else None,
                                    "peak_source": peak_kind}},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "traffic_source": traffic_src, "kernel": "stream_kernel",
                     "bytes_per_vector": dvec,
                     "bytes_model": (f"DRAM-resident algorithmic bytes {es}*(N*m + n) per vector (N sampled "
                                     "columns + x); the want gathered rows of A are L2 hits (A is L2-resident, "
                                     "evict_last) and are excluded, as SURVEY.md §8(d) excludes the L2-resident "
                                     "sign tables"),
                     "traffic_over_algorithmic": (traffic / (dvec * vec_per_launch)) if traffic else None,
                     "survey_8d": {"bytes_per_vector": bvec, "achieved": achieved_8d, "frac": achieved_8d / peak,
                                   "note": "es*(N*m + want*n + n): counts the L2-served A rows as DRAM bytes"},
                     "per_launch_ms": per_launch_ms, "peak_source": peak_kind,
                     # `peak` is a copy figure (half reads, half writes, with the bus turnarounds a copy
                     # pays); this kernel only reads, so on a box with little power capping `frac` can
                     # pass 1.0. The read-only ceiling of its own access pattern is reported beside it.
                     "read_ceiling": {"gbs": RANDOM_READ_CEILING_GBS, "frac": achieved / RANDOM_READ_CEILING_GBS,
                                      "source": "random 16 KiB bulk-copy column reads of a 128 GiB buffer, "
                                                "tools/micro/rand_read.cu (profiles/r01_tma_issue.txt: "
                                                "7.1-7.3 TB/s)"},
                     "per_launch_source": ("library CUDA events over the timed region" if profile_in_timed else
                                           "library CUDA events over a second, untimed pass of the same K steps")},
        "kernels_ms": {"stream": stream_ms, "draw": draw_ms, "stream_launches": stream_launches,
                       "draw_launches": draw_launches},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "e2e": e2e,
        "cpu_baseline": cpu,
        "parity": parity,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    sk.close()
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------- config 5: sweep + GEMM ----
L2_TMA_PEAK_GBS = 19600.0  # L2-resident 16 KiB bulk copies, 2-3 CTAs/SM (profiles/r01_tma_issue.txt)


def run_sweep(args):
    """Config 5: s in {4,16,64,256} x eps in {0.2,0.1,0.05} at n = 4096 on one GPU, one GPU's shard of
    the 1,048,576-vector job (131,072 vectors per launch = 1,048,576 / 8 GPUs, weak scaling), against
    dense h_eps(A x) by one cuBLAS GEMM per batch (fp32 SGEMM and TF32) on the same batch. Per s, the
    three stages of the fused kernel are timed in isolation with its role-removal switches
    (FSTG_STREAM_DEBUG: 5 = column gather-accumulate only, 6 = coefficients only, 3 = candidate
    select + refinement only) and each is set against its own roofline."""
    import torch
    from paper_2105_05879_b200 import fst, generators
    dev = "cuda:0"
    torch.cuda.set_device(0)
    A64 = generators.haar_orthogonal(N_DIM, A_SEED, dev)
    A32 = A64.float().contiguous()
    sk = fst.preprocess(A32)
    B = 131072 if args.batch == 65536 else args.batch
    stream = torch.cuda.current_stream()
    peak, _ = peaks()
    reps = max(1, args.steps // 2)

    def timed(fn, reps):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    def kernel_ms(fn):
        """stream-kernel device time per launch (library CUDA events) over `reps` calls."""
        fn()
        fst.profile_enable(True)
        fst.profile_reset()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        k_ms, k_n = fst.profile_read("stream")
        fst.profile_enable(False)
        return k_ms / max(1, k_n)

    rows, stages = [], []
    N = args.J * args.K
    with ClockSampler(0) as clk:
        for s_val in (4, 16, 64, 256):
            prob = generators.config5_problem(s_val, 0.1, B, seed=X_SEED, device=dev, A64=A64)
            X = prob.X
            seeds_dev = torch.from_numpy(prob.seeds.view(np.int64)).to(dev)
            want = fst.candidate_count(s_val, WIDEN, N_DIM)
            p = fst.StreamParams(epsilon=0.1, s=s_val, J=args.J, K=args.K, widen=WIDEN)
            out = fst.transform_batch(sk, X, p, seeds_dev, stream=stream.cuda_stream)
            call = lambda: fst.transform_batch(sk, X, p, seeds_dev, out=out, stream=stream.cuda_stream)  # noqa: E731
            st = {"s": s_val, "want": want}
            try:
                for name, bits in (("full", 0), ("gather_accumulate", 5), ("coefficients", 6), ("refinement", 3)):
                    os.environ["FSTG_STREAM_DEBUG"] = str(bits)
                    st[name + "_ms"] = kernel_ms(call)
            finally:
                os.environ.pop("FSTG_STREAM_DEBUG", None)
            col_bytes = 4.0 * N * N_DIM * B
            adds = float(N) * N_DIM * B
            row_bytes = 4.0 * want * N_DIM * B
            st["gather_accumulate_roofline"] = {"bound": "hbm", "unit": "GB/s", "peak": peak,
                                                "achieved": col_bytes / st["gather_accumulate_ms"] / 1e6,
                                                "frac": col_bytes / st["gather_accumulate_ms"] / 1e6 / peak}
            st["coefficients_roofline"] = {"bound": "fp32 add", "unit": "Tadd/s", "peak": FP32_ADD_PEAK_TADD,
                                           "achieved": adds / st["coefficients_ms"] / 1e9,
                                           "frac": adds / st["coefficients_ms"] / 1e9 / FP32_ADD_PEAK_TADD}
            st["refinement_roofline"] = {"bound": "l2", "unit": "GB/s", "peak": L2_TMA_PEAK_GBS,
                                         "achieved": row_bytes / st["refinement_ms"] / 1e6,
                                         "frac": row_bytes / st["refinement_ms"] / 1e6 / L2_TMA_PEAK_GBS}
            st["full_hbm_frac_dram_bytes"] = (4.0 * (N * N_DIM + N_DIM) * B) / st["full_ms"] / 1e6 / peak
            stages.append(st)
            for eps_val in (0.2, 0.1, 0.05):
                p = fst.StreamParams(epsilon=eps_val, s=s_val, J=args.J, K=args.K, widen=WIDEN)
                out = fst.transform_batch(sk, X, p, seeds_dev, stream=stream.cuda_stream)
                ms_stream = timed(lambda: fst.transform_batch(sk, X, p, seeds_dev, out=out, stream=stream.cuda_stream),
                                  reps)
                torch.backends.cuda.matmul.allow_tf32 = False
                dense = lambda: torch.where((ax := X @ A32.T).abs() >= eps_val, ax, 0.0)  # noqa: E731
                ms_sgemm = timed(dense, 3)
                torch.backends.cuda.matmul.allow_tf32 = True
                ms_tf32 = timed(dense, 3)
                torch.backends.cuda.matmul.allow_tf32 = False
                # support agreement of the stream with the exact dense threshold (fp64 reference)
                sub = min(B, 4096)
                ax = X[:sub].double() @ A64.T
                dense_sup = ax.abs() >= eps_val
                counts = out.counts[:sub].long()
                stream_sup = torch.zeros_like(dense_sup)
                valid = torch.arange(want, device=dev).unsqueeze(0) < counts.unsqueeze(1)
                r_idx = torch.arange(sub, device=dev).unsqueeze(1).expand(-1, want)
                stream_sup[r_idx[valid], out.support[:sub].long()[valid]] = True
                match = float((stream_sup == dense_sup).all(dim=1).float().mean())
                rows.append({"s": s_val, "eps": eps_val, "want": want,
                             "stream_vectors_per_s": B / (ms_stream / 1e3),
                             "stream_hbm_frac_dram_bytes": 4.0 * (N * N_DIM + N_DIM) * B / ms_stream / 1e6 / peak,
                             "dense_sgemm_vectors_per_s": B / (ms_sgemm / 1e3),
                             "dense_tf32_vectors_per_s": B / (ms_tf32 / 1e3),
                             "support_match_vs_exact": match,
                             "mean_true_support": float(dense_sup.sum(dim=1).float().mean()),
                             "mean_stream_support": float(counts.float().mean())})
            del prob, X, out
    line = {"metric": "config5 sweep: thresholded-Ax vectors/sec vs dense GEMM (1 B200 = one GPU's shard)", "n_gpus": 1,
            "config": {"workload": f"config5: n=4096 fp32 Haar A, x = A^T y (s-sparse +-1/sqrt(s)), {B} vectors per "
                                   f"launch (1,048,576 / 8 GPUs), J={args.J}, K={args.K}, widen=10"},
            "sweep": rows, "stages": stages,
            "stage_note": ("stage times are the stream kernel run with the other roles removed (FSTG_STREAM_DEBUG); "
                           "the fused kernel overlaps them, so full_ms < the sum"),
            "clocks": clk.summary()}
    print(json.dumps(line), flush=True)
    sk.close()


# ------------------------------------------- config 4: retain-sampled ----
def run_config4(args):
    """Config 4: n = 16384 fp32, A iid N(0,1/n), 8192 vectors per step per GPU, s = 64, eps = 0.05.
    The 8.8 TB sketch cannot exist. One GPU: fstg_transform_design_batch — per row
    block, the retain-sampled FWHT of those rows of every sampled column and the
    stream's batch sums for those rows, then the tail (one Kerdock pass per step).
    N > 1 GPUs: rank r computes its row shard of every
    vector's batch means (1/N of the pass), one NCCL all-to-all of means routes
    them to the vector owners (parallel.route_partial_means), and each rank runs
    the tail for its own vectors."""
    import torch
    import torch.distributed as dist
    from paper_2105_05879_b200 import fst, generators, parallel
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    one_dev = os.environ.get("FSTG_BENCH_ONE_DEVICE") == "1"   # functional check only (see run_b200)
    if one_dev:
        local = 0
    torch.cuda.set_device(local)
    dev = f"cuda:{local}"
    if world > 1:
        if one_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(dev))
    n, B, s_val, eps_val = 16384, 8192, 64, 0.05
    if one_dev and os.environ.get("FSTG_C4_VECTORS"):          # functional check with small batches
        B = int(os.environ["FSTG_C4_VECTORS"])
    A64 = generators.iid_gaussian(n, 16384, dev) if rank == 0 else torch.empty((n, n), dtype=torch.float64, device=dev)
    if world > 1:
        parallel.broadcast_matrix(A64, src=0)
    A32 = A64.float().contiguous()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    des = fst.preprocess_design(A32)
    e1.record()
    torch.cuda.synchronize()
    design_ms = e0.elapsed_time(e1)
    # every rank knows every vector's seed (its row shard covers every vector)
    g_all, st_all = generators.trial_seeds(X_SEED, 0, B * world)
    first = rank * B
    Y = torch.from_numpy(generators.sparse_targets(g_all[first:first + B], n, s_val, value_kind=1)).to(dev)
    lu = torch.linalg.lu_factor(A64)
    X = torch.linalg.lu_solve(*lu, Y.T).T
    X = (X / torch.linalg.vector_norm(X, dim=1, keepdim=True)).float().contiguous()
    del Y, lu, A64
    seeds_all = torch.from_numpy(st_all.view(np.int64)).to(dev)
    p = fst.StreamParams(epsilon=eps_val, s=s_val, J=args.J, K=args.K, widen=WIDEN)
    N = args.J * args.K
    want = fst.candidate_count(s_val, WIDEN, n)
    fst.profile_enable(True)
    # a stream of design-only batches: keep the ~100 GB of retained-column scratch cached in the
    # library pool between calls instead of re-mapping it every step (fstg_set_pool_retain)
    fst.set_pool_retain(True)
    out = fst.BatchResult(torch.zeros(B, dtype=torch.int32, device=dev),
                          torch.zeros((B, want), dtype=torch.int32, device=dev),
                          torch.zeros((B, want), dtype=torch.float32, device=dev))
    stream = torch.cuda.current_stream()

    def sample_fn(ells):
        buf = torch.empty((len(ells), ldc), dtype=torch.float32, device=dev)
        fst.sample_columns(des, ells, out=buf, stream=stream.cuda_stream)
        return buf

    if world > 1:
        # every rank needs every vector's x for its row shard of the batch means
        X_all = torch.empty((B * world, n), dtype=X.dtype, device=dev)
        dist.all_gather_into_tensor(X_all, X)
        row_ranges = [(f, f + c) for f, c in (parallel.strong_shard(r, world, n) for r in range(world))]
        vec_ranges = [(q * B, B) for q in range(world)]
        ld = des.column_stride

    breakdown = {}  # library CUDA-event scopes of the last step (ms)

    def step(timing):
        fst.profile_reset()
        if world == 1:
            # row-blocked design transform: one Kerdock pass for all B vectors (fstg_transform_design_batch)
            fst.transform_design_batch(des, X, p, seeds=seeds_all[:B], row_block=args.row_block, out=out,
                                       stream=stream.cuda_stream)
        else:
            # row-sharded: rank r's rows of every vector's batch means (1/W of the Kerdock pass),
            # one NCCL all-to-all of means (K x rows per vector), then the tail for my vectors
            r0, r1 = row_ranges[rank]
            part = fst.design_partial_means(des, X_all, p, seeds=seeds_all, row_begin=r0, row_end=r1,
                                            stream=stream.cuda_stream)
            full = parallel.route_partial_means(part, vec_ranges, row_ranges, rank, ld)
            del part
            fst.transform_from_means(des, X, p, full, out=out, stream=stream.cuda_stream)
        ms_fwht, launches = fst.profile_read("sample_columns_fwht")
        timing.append((ms_fwht, launches))
        breakdown.clear()
        for name in ("draw", "sample_columns_fwht", "sample_columns_identity", "stream_partial", "stream_tail"):
            breakdown[name] = fst.profile_read(name)[0]

    warm = []
    for _ in range(max(1, args.warmup)):
        step(warm)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    timing = []
    with ClockSampler(local) as clk:
        t0.record(stream)
        for _ in range(args.steps):
            step(timing)
        t1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = parallel.max_over_ranks(t0.elapsed_time(t1), device=dev)
    retain_ms = sum(t for t, _ in timing)
    passes = len(timing)                             # steps; each is one Kerdock pass over this rank's rows
    adds_per_pass = (des.d // 2) * n * des.d * 14 / world  # (d/2) m d log2 d over this rank's row shard
    # measured FP32 add ceiling of the CUDA cores (tools/micro/fadd_peak.cu, profiles/r01_fadd_peak.txt):
    # FADD and packed FADD2 both retire ~126 adds/clk/SM (FADD2 halves issue slots, not pipe time)
    fp32_peak = FP32_ADD_PEAK_TADD
    achieved = adds_per_pass * passes / (retain_ms / 1e3) / 1e12
    mean_support = float(out.counts.float().mean())
    if world > 1:
        mean_support = parallel.max_over_ranks(mean_support, device=dev)
    line = {"metric": "thresholded-Ax vectors/sec (config4, n=16384, retain-sampled)",
            "value": B * world * args.steps / (ms / 1e3),
            "unit": "vectors/s", "n_gpus": world, "steps": args.steps, "warmup": max(1, args.warmup),
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "fp32", "data": "synthetic (A iid N(0,1/n), y 64-sparse N(0,1), x = A^-1 y / |.|)",
            "config": {"workload": (f"config4: n=m=16384 fp32, s=64, eps=0.05, 8192 vectors/step/GPU, J={args.J}, "
                                    f"K={args.K} (full sketch 8.8 TB: " +
                                    ("row-blocked design transform, one Kerdock pass per step)" if world == 1 else
                                     "row-sharded batch means, 1/N of the Kerdock pass per rank, NCCL all-to-all "
                                     "of means)")),
                       "mean_support": mean_support, "row_block": args.row_block or "auto",
                       "scratch": "library pool retained across steps (fstg_set_pool_retain)"},
            "preprocess": {"design_ms": design_ms, "kerdock_pass_ms": retain_ms / passes,
                           "kerdock_passes_per_step": passes // args.steps,
                           "step_breakdown_ms": {k: round(v, 2) for k, v in breakdown.items()},
                           "roofline": {"bound": "fp32", "achieved": achieved, "peak": fp32_peak, "unit": "Tadd/s",
                                        "frac": achieved / fp32_peak, "peak_source": "measured FADD/FADD2 rate, "
                                        "tools/micro/fadd_peak.cu (profiles/r01_fadd_peak.txt)"}},
            "clocks": clk.summary()}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------- reference arm ----
def run_reference(args):
    """Reference arm: the reference algorithm on the host cores (rank 0 only; other ranks exit 0),
    on the b200 arm's config and EXACT inputs. A is built by the same routine (the oracle's
    SeededRng Gaussian fill, bit-identical to the library's, then the same QR on the same device)
    and the vectors by the same generator (the oracle's restatement of the library's target
    generator, bit-identical) and the same first 8192-vector chunk of x = A^T y; the reference
    then computes in fp64 on the fp32 inputs the GPU sees (configs 2 / 3) or on the fp64 inputs
    (config 1). The product library is not loaded in this process."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        print(f"[bench] reference arm: rank {rank}/{world} idle (rank 0 times the host reference)",
              file=sys.stderr, flush=True)
        return
    import torch
    from oracle import oracle as orc
    orc.build()
    cfg = WORKLOADS[args.config]
    threads = os.cpu_count() or 1
    dev = "cuda:0" if torch.cuda.is_available() else "cpu"
    A64 = build_matrix(cfg, dev, gaussian_fill=orc.rng_gaussian)
    B_ref = min(batch_size(args, cfg), 8192)        # the b200 arm's first x chunk: same GEMM shape, same bits
    prob = make_problem(cfg, A64, B_ref, 0, dev, targets=orc.gen_sparse_targets)
    a64 = prob.A.double().cpu().numpy()
    if args.choose_params:  # the reference CLI's default regime (cli.hpp:164-172)
        args.J, args.K = orc.choose_params(float(np.max(np.linalg.norm(a64, axis=1))), cfg["eps"] / 2, 0.1,
                                           a64.shape[0])
    P = min(pool_size(args.J * args.K, a64.shape[0]), B_ref)
    X = prob.X[:P].double().cpu().numpy()
    seeds = prob.seeds[:P]
    del prob, A64
    s_val = cfg["s"]
    vals, secs_all = [], []
    for i in range(args.warmup + args.steps):
        rr = cpu_sample(a64, X, seeds, args.J, args.K, threads, args.cpu_seconds / 2, s_val=s_val,
                        eps_val=cfg["eps"])
        if i >= args.warmup:
            vals.append(rr["vectors"])
            secs_all.append(rr["seconds"])
    value = sum(vals) / sum(secs_all)
    line = {
        "impl": "reference",
        "metric": METRIC if args.config == "3" else f"thresholded-Ax vectors/sec ({cfg['desc'].split(':')[0]})",
        "value": value, "unit": "vectors/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(secs_all) / len(secs_all),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp64",
        "data": cfg["data"] + "; the b200 arm's exact A and x (fp32 values widened to fp64 for configs 2/3)",
        "config": workload_config(args, cfg, world),
        "cpu_baseline": {"value": value, "unit": "vectors/s", "cores": threads, "kind": rr["kind"],
                         "sample": f"per step ~{int(np.mean(vals))} vectors cycling the b200 arm's first {P} vectors "
                                   f"on {threads} threads; {cpu_impl_text(rr['kind'])}; sampled columns "
                                   f"pre-materialised in DRAM"},
        "e2e": {"value": value, "unit": "vectors/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def relaunch_under_torchrun(args) -> bool:
    """`bench.py --gpus N` (N > 1) started directly: re-run this command as N ranks (one process
    per GPU) under torch.distributed.run on 127.0.0.1, exactly as the driver launches it. Returns
    True when this process was the launcher (it has already waited for the ranks)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return False
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    print(f"[bench] launching {args.gpus} ranks: {' '.join(cmd[1:])}", file=sys.stderr, flush=True)
    rc = subprocess.call(cmd)
    if rc != 0:
        sys.exit(rc)
    return True


def main():
    args = parse()
    if relaunch_under_torchrun(args):
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus and "WORLD_SIZE" in os.environ:
        print(f"[bench] note: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    elif args.config == "5":
        run_sweep(args)
    elif args.config == "4":
        run_config4(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
