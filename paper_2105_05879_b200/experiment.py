"""GPU experiment harness — reference experiment.hpp:109-219 on the B200 path.

Same config keys (`n s trials Jgrid Kgrid epsilon delta widen seed p sketch
mode`), same per-trial seed schedule (trial_seed = seed ^ trial; x from
gen_seed(trial_seed), indices from stream_seed(trial_seed)), same generators
(gen_exact_sparse / gen_mixture draw order, generators.hpp:38-85), same
outputs: per (J, K) the worst |mu - Ax|_inf, the worst |h - h_eps(Ax)|_2 over
the trials and the streaming / naive runtime ratio, and the same CSV.

Differences by design: all trials of a grid point run as ONE batched
transform (the whole point of the GPU path), the naive product is the batched
dense GEMM A X^T on the same device (cuBLAS via torch, fp64 for the error
reference, plus an fp32 SGEMM timing for the crossover), and times are CUDA
events instead of steady_clock. Like the reference, index draws and column
fetches are part of the streaming time only in `timing="e2e"` mode; the
default "kernel" mode times the transform launch (draw + stream kernels).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import fst, generators


@dataclass
class ExperimentConfig:
    """experiment.hpp:111-132"""
    n: int = 256
    s: int = 20
    trials: int = 100
    j_grid: List[int] = field(default_factory=list)
    k_grid: List[int] = field(default_factory=list)
    epsilon: float = 0.1
    delta: float = 0.0
    widen: int = 10
    seed: int = 0
    mode: str = "exact-sparse"      # or "gaussian-mixture"
    mixture_p: float = 0.05
    sketch_path: str = ""

    def validate(self) -> None:
        if self.n < 1:
            raise ValueError("ExperimentConfig: n must be positive")
        if self.trials < 0:
            raise ValueError("ExperimentConfig: trials must be >= 0")
        if not self.j_grid or not self.k_grid:
            raise ValueError("ExperimentConfig: parameter grids must be nonempty")


@dataclass
class ExperimentRow:
    """experiment.hpp:134-140"""
    J: int
    K: int
    worst_inf_err: float = 0.0
    worst_l2_err: float = 0.0
    runtime_ratio: float = 0.0
    stream_ms: float = 0.0
    naive_ms: float = 0.0


def parse_config(text: str) -> ExperimentConfig:
    """experiment.hpp:165-199: flat key=value, '#' comments."""
    cfg = ExperimentConfig()
    for raw in text.splitlines():
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise ValueError(f"config: expected key=value, got '{line}'")
        key, value = (t.strip() for t in line.split("=", 1))
        ints = lambda v: [int(t) for t in v.split(",") if t.strip()]  # noqa: E731
        if key == "n":
            cfg.n = int(value)
        elif key == "s":
            cfg.s = int(value)
        elif key == "trials":
            cfg.trials = int(value)
        elif key == "Jgrid":
            cfg.j_grid = ints(value)
        elif key == "Kgrid":
            cfg.k_grid = ints(value)
        elif key == "epsilon":
            cfg.epsilon = float(value)
        elif key == "delta":
            cfg.delta = float(value)
        elif key == "widen":
            cfg.widen = int(value)
        elif key == "seed":
            cfg.seed = int(value)
        elif key == "p":
            cfg.mixture_p = float(value)
        elif key == "sketch":
            cfg.sketch_path = value
        elif key == "mode":
            if value not in ("exact-sparse", "gaussian-mixture"):
                raise ValueError(f"config: unknown mode '{value}'")
            cfg.mode = value
        else:
            raise ValueError(f"config: unknown key '{key}'")
    return cfg


def trial_inputs(A64, cfg: ExperimentConfig):
    """x for trials 0..T-1 (experiment.hpp:163-167) and their stream seeds; fp64 torch on A64's device."""
    import torch
    t = np.uint64(cfg.seed) ^ np.arange(cfg.trials, dtype=np.uint64)
    gen = generators.mix_seed(t ^ np.uint64(generators.GEN_TAG))
    st = generators.mix_seed(t ^ np.uint64(generators.TRX_TAG))
    m = A64.shape[0]
    if cfg.mode == "exact-sparse":
        Y = generators.sparse_targets(gen, m, cfg.s)
        X = torch.from_numpy(Y).to(A64.device) @ A64                       # x = A^T y
    else:
        Y = np.empty((cfg.trials, m), dtype=np.float64)
        g = np.ascontiguousarray(gen, dtype=np.uint64)
        fst._check(fst.lib().fstg_gen_mixture_targets(g.ctypes.data_as(C.c_void_p), C.c_int64(cfg.trials),
                                                       C.c_int64(m), C.c_double(cfg.mixture_p),
                                                       Y.ctypes.data_as(C.c_void_p)))
        X = torch.from_numpy(Y).to(A64.device) @ A64
        X = X / torch.linalg.vector_norm(X, dim=1, keepdim=True)
    return X.contiguous(), st


def run_experiment(cfg: ExperimentConfig, sk: fst.Sketch, A64) -> List[ExperimentRow]:
    """experiment.hpp:231-289 with batched trials. A64: the sketch's matrix (torch fp64, cuda)."""
    import torch
    cfg.validate()
    if sk.n != cfg.n:
        raise ValueError("run_experiment: sketch n does not match the config")
    rows: List[ExperimentRow] = []
    if cfg.trials == 0:
        return rows
    X64, seeds = trial_inputs(A64, cfg)
    Xs = X64.to(torch.float64 if sk.dtype == np.float64 else torch.float32).contiguous()
    seeds_d = torch.from_numpy(seeds.view(np.int64)).to(X64.device)
    ax = X64 @ A64.T                                                          # (T, m): naive Ax, fp64
    h_ref = torch.where(ax.abs() >= cfg.epsilon, ax, torch.zeros_like(ax))
    A_c = A64.to(Xs.dtype)
    stream = torch.cuda.current_stream()
    for J in cfg.j_grid:
        for K in cfg.k_grid:
            p = fst.StreamParams(epsilon=cfg.epsilon, delta=cfg.delta, s=cfg.s, J=J, K=K, widen=cfg.widen)
            out = fst.transform_batch(sk, Xs, p, seeds_d, mu=True, stream=stream.cuda_stream)
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(stream)
            fst.transform_batch(sk, Xs, p, seeds_d, out=out, stream=stream.cuda_stream)
            e1.record(stream)
            dense = Xs @ A_c.T                                                # the naive product, same batch
            e2.record(stream)
            torch.cuda.synchronize()
            del dense
            stream_ms, naive_ms = e0.elapsed_time(e1), e1.elapsed_time(e2)
            mu = out.mu.to(torch.float64)
            inf_err = float((mu - ax).abs().max(dim=1).values.max())
            h = torch.zeros_like(ax)
            counts = out.counts.long()
            want = out.support.shape[1]
            valid = torch.arange(want, device=ax.device).unsqueeze(0) < counts.unsqueeze(1)
            rows_i = torch.arange(cfg.trials, device=ax.device).unsqueeze(1).expand(-1, want)
            h[rows_i[valid], out.support.long()[valid]] = out.values.to(torch.float64)[valid]
            l2_err = float(torch.linalg.vector_norm(h - h_ref, dim=1).max())
            rows.append(ExperimentRow(J, K, inf_err, l2_err, stream_ms / naive_ms if naive_ms > 0 else 0.0,
                                      stream_ms, naive_ms))
    return rows


def to_csv(rows: List[ExperimentRow]) -> str:
    """experiment.hpp:296-306 (same columns, %.17g)."""
    out = ["J,K,worst_inf_err,worst_l2_err,runtime_ratio"]
    for r in rows:
        out.append(f"{r.J},{r.K},{r.worst_inf_err:.17g},{r.worst_l2_err:.17g},{r.runtime_ratio:.17g}")
    return "\n".join(out) + "\n"


def dense_threshold(A, X, eps: float):
    """The dense alternative: h_eps(A x) for a batch by one GEMM (cuBLAS) + threshold.
    Returns (values (B, m) with zeros below eps)."""
    import torch
    ax = X @ A.T
    return torch.where(ax.abs() >= eps, ax, torch.zeros_like(ax))
