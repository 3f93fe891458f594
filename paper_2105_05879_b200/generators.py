"""Seeded synthetic inputs for the BASELINE.json configurations (product side).

Conventions follow the reference harness: SeededRng streams (rng.hpp) via the
library's host generators, gen_orthogonal's Gaussian fill + QR with
sign-corrected R diagonal (generators.hpp:20-33), gen_exact_sparse's draw
order (generators.hpp:38-55), and the per-trial seed schedule of
experiment.hpp:133-136 (trial_seed = seed ^ v; x from mix_seed(t ^ "gen"),
indices from mix_seed(t ^ "trx")), so vector v's inputs do not depend on the
GPU count or batch split. QR / solve / A^T y run in fp64 on the GPU via torch
(cuSOLVER/cuBLAS: input plumbing, not the measured path).

configs (BASELINE.json):
  1  n=256  fp64, A Haar orthogonal, y s=8 +-1/sqrt(8),                x = A^T y, eps 0.1
  2  n=1024 fp32, A iid N(0,1/n),    y s=16 N(0,1) values,             x = A^-1 y / |.|, eps 0.05
  3  n=4096 fp32, A Haar orthogonal, y s=32 +-1/sqrt(32) + N(0,1e-6),  x = A^T y / |.|, eps 0.1
  5  n=4096 fp32, A Haar orthogonal, y s in {4,16,64,256} +-1/sqrt(s), x = A^T y,       eps in {0.2,0.1,0.05}
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import fst

_M64 = (1 << 64) - 1
GEN_TAG = 0x67656E   # "gen"
TRX_TAG = 0x747278   # "trx"


def mix_seed(z):
    """SplitMix64 step (rng.hpp:54-59), vectorised over uint64 arrays."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def trial_seeds(seed: int, first: int, count: int):
    """experiment.hpp:133-136,163: (generator seeds, stream seeds) of vectors first..first+count."""
    t = np.uint64(seed) ^ np.arange(first, first + count, dtype=np.uint64)
    return mix_seed(t ^ np.uint64(GEN_TAG)), mix_seed(t ^ np.uint64(TRX_TAG))


def gaussian(seed: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.float64)
    fst._check(fst.lib().fstg_gen_gaussian(C.c_uint64(seed), C.c_int64(count), out.ctypes.data_as(C.c_void_p)))
    return out


def sparse_targets(gen_seeds: np.ndarray, m: int, s: int, value_kind: int = 0, noise_sigma: float = 0.0):
    gen_seeds = np.ascontiguousarray(gen_seeds, dtype=np.uint64)
    Y = np.empty((len(gen_seeds), m), dtype=np.float64)
    fst._check(fst.lib().fstg_gen_sparse_targets(gen_seeds.ctypes.data_as(C.c_void_p), C.c_int64(len(gen_seeds)),
                                                 C.c_int64(m), C.c_int64(s), C.c_int(value_kind),
                                                 C.c_double(noise_sigma), Y.ctypes.data_as(C.c_void_p)))
    return Y


def haar_orthogonal(n: int, seed: int, device="cuda:0", gaussian_fill=None):
    """generators.hpp:20-33 on the GPU (fp64): QR of the SeededRng Gaussian fill, diag(R) > 0.
    gaussian_fill(seed, count) replaces the library's fill (bench.py's reference arm passes the
    oracle's bit-identical SeededRng so that it does not load the product library)."""
    import torch
    g = torch.from_numpy((gaussian_fill or gaussian)(seed, n * n).reshape(n, n)).to(device)
    q, r = torch.linalg.qr(g)
    sign = torch.sign(torch.diagonal(r))
    sign[sign == 0] = 1
    return q * sign.unsqueeze(0)


def iid_gaussian(n: int, seed: int, device="cuda:0", gaussian_fill=None):
    import torch
    return torch.from_numpy((gaussian_fill or gaussian)(seed, n * n).reshape(n, n)).to(device) / np.sqrt(n)


@dataclass
class Problem:
    name: str
    A: object              # torch (m, n), compute dtype, on device
    X: object              # torch (B, n), compute dtype, on device
    seeds: np.ndarray      # per-vector stream seeds (uint64)
    eps: float
    s: int
    dtype: object
    A64: object = None     # fp64 copy of A (torch, device)


def _apply(A64, Y, mode: str, normalize: bool, chunk: int = 8192):
    """x = A^T y (mode 'T') or A^{-1} y (mode 'inv'), optionally unit-normalised, fp64, chunked."""
    import torch
    out = []
    lu = None
    for c0 in range(0, Y.shape[0], chunk):
        y = torch.from_numpy(Y[c0:c0 + chunk]).to(A64.device)
        if mode == "T":
            x = y @ A64                      # (A^T y)^T = y^T A
        else:
            if lu is None:
                lu = torch.linalg.lu_factor(A64)
            x = torch.linalg.lu_solve(*lu, y.T).T
        if normalize:
            x = x / torch.linalg.vector_norm(x, dim=1, keepdim=True)
        out.append(x)
    return torch.cat(out, 0)


def config1_problem(B: int = 64, seed: int = 0, device="cuda:0", a_seed: int = 777, targets=None,
                    A64=None) -> Problem:
    import torch
    if A64 is None:
        A64 = haar_orthogonal(256, a_seed, device)
    g, st = trial_seeds(seed, 0, B)
    X = _apply(A64, (targets or sparse_targets)(g, 256, 8), "T", False)
    return Problem("config1", A64, X.to(torch.float64), st, 0.1, 8, torch.float64, A64)


def config2_problem(B: int = 4096, seed: int = 0, device="cuda:0", a_seed: int = 1024, first: int = 0,
                    targets=None, A64=None) -> Problem:
    import torch
    if A64 is None:
        A64 = iid_gaussian(1024, a_seed, device)
    g, st = trial_seeds(seed, first, B)
    X = _apply(A64, (targets or sparse_targets)(g, 1024, 16, value_kind=1), "inv", True)
    return Problem("config2", A64.float().contiguous(), X.float().contiguous(), st, 0.05, 16, torch.float32, A64)


def config3_problem(B: int = 65536, seed: int = 0, device="cuda:0", a_seed: int = 4096, first: int = 0,
                    A64=None, targets=None) -> Problem:
    import torch
    if A64 is None:
        A64 = haar_orthogonal(4096, a_seed, device)
    g, st = trial_seeds(seed, first, B)
    X = _apply(A64, (targets or sparse_targets)(g, 4096, 32, value_kind=0, noise_sigma=1e-3), "T", True)
    return Problem("config3", A64.float().contiguous(), X.float().contiguous(), st, 0.1, 32, torch.float32, A64)


def config5_problem(s: int, eps: float, B: int, seed: int = 0, device="cuda:0", a_seed: int = 4096, first: int = 0,
                    A64=None) -> Problem:
    import torch
    if A64 is None:
        A64 = haar_orthogonal(4096, a_seed, device)
    g, st = trial_seeds(seed, first, B)
    X = _apply(A64, sparse_targets(g, 4096, s), "T", False)
    return Problem(f"config5_s{s}_eps{eps}", A64.float().contiguous(), X.float().contiguous(), st, eps, s,
                   torch.float32, A64)
