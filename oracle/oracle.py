"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes front-end over ``oracle/libfst_oracle.so`` (the Eigen-free C++
restatement of /root/reference/proj/include/fst, see fst_oracle.hpp). Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may import
this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

from typing import NamedTuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libfst_oracle.so")
_lib = None

class IoError(OSError):
    pass


class MagicMismatchError(IoError):
    pass


class VersionUnsupportedError(IoError):
    pass


class TruncatedPayloadError(IoError):
    pass


class MalformedHeaderError(IoError):
    pass


_ERRORS = {1: ValueError, 2: IndexError, 3: OverflowError, 4: RuntimeError, 5: RuntimeError, 7: IoError,
           8: MagicMismatchError, 9: VersionUnsupportedError, 10: TruncatedPayloadError, 11: MalformedHeaderError}


def build() -> str:
    """Compile the restatement (g++, -ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        _lib.orc_last_error.restype = C.c_char_p
        _lib.orc_coords_of_position.restype = C.c_uint64
        _lib.orc_position_of_coords.restype = C.c_uint64
        _lib.orc_mix_seed.restype = C.c_uint64
        _lib.orc_gen_seed.restype = C.c_uint64
        _lib.orc_stream_seed.restype = C.c_uint64
        _lib.orc_mix_seed.argtypes = [C.c_uint64]
        _lib.orc_gen_seed.argtypes = [C.c_uint64]
        _lib.orc_stream_seed.argtypes = [C.c_uint64]
        _lib.orc_candidate_count.restype = C.c_int64
        _lib.orc_candidate_count.argtypes = [C.c_int64, C.c_int64, C.c_int64]
        _lib.orc_sketch_columns.restype = C.c_void_p
        _lib.orc_sketch_columns.argtypes = [C.c_void_p]
        _lib.orc_sketch_free.argtypes = [C.c_void_p]
        _lib.orc_design_moment_target.restype = C.c_double
        _lib.orc_design_moment_target.argtypes = [C.c_int64, C.c_int]
    return _lib


def _check(rc: int) -> None:
    if rc != 0:
        raise _ERRORS.get(rc, RuntimeError)(lib().orc_last_error().decode())


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ------------------------------------------------------------------ gf2 ----
def modulus_for_degree(q: int) -> int:
    out = C.c_uint64()
    _check(lib().orc_modulus_for_degree(C.c_int(q), C.byref(out)))
    return out.value


def verify_irreducible(poly: int, degree: int) -> bool:
    out = C.c_int()
    _check(lib().orc_verify_irreducible(C.c_uint64(poly), C.c_int(degree), C.byref(out)))
    return bool(out.value)


def field_mul(q: int, a: int, b: int) -> int:
    out = C.c_uint64()
    _check(lib().orc_field_mul(C.c_int(q), C.c_uint64(a), C.c_uint64(b), C.byref(out)))
    return out.value


def field_trace(q: int, a: int) -> int:
    out = C.c_int()
    _check(lib().orc_field_trace(C.c_int(q), C.c_uint64(a), C.byref(out)))
    return out.value


def gf2_rank(rows) -> int:
    arr = np.ascontiguousarray(rows, dtype=np.uint64)
    return lib().orc_gf2_rank(_ptr(arr), C.c_int(len(arr)))


def coords_of_position(p: int, k: int) -> int:
    return lib().orc_coords_of_position(C.c_uint64(p), C.c_int(k))


def position_of_coords(w: int, k: int) -> int:
    return lib().orc_position_of_coords(C.c_uint64(w), C.c_int(k))


# -------------------------------------------------------------- kerdock ----
def design_params(k: int):
    d, L = C.c_int64(), C.c_int64()
    _check(lib().orc_design_params(C.c_int(k), C.byref(d), C.byref(L)))
    return d.value, L.value


def kerdock_matrix(k: int, s: int) -> np.ndarray:
    out = np.zeros(k, dtype=np.uint64)
    _check(lib().orc_kerdock_matrix(C.c_int(k), C.c_uint64(s), _ptr(out)))
    return out


def quadratic_form(rows, x: int) -> int:
    arr = np.ascontiguousarray(rows, dtype=np.uint64)
    return lib().orc_quadratic_form(_ptr(arr), C.c_int(len(arr)), C.c_uint64(x))


def reversed_q_rows(rows) -> np.ndarray:
    arr = np.ascontiguousarray(rows, dtype=np.uint64)
    out = np.zeros(len(arr), dtype=np.uint64)
    lib().orc_reversed_q_rows(_ptr(arr), C.c_int(len(arr)), _ptr(out))
    return out


def decode_index(k: int, ell: int):
    ident, s, w = C.c_int(), C.c_uint64(), C.c_uint64()
    _check(lib().orc_decode_index(C.c_int(k), C.c_int64(ell), C.byref(ident), C.byref(s), C.byref(w)))
    return bool(ident.value), s.value, w.value


def projected_design_column(k: int, n: int, ell: int) -> np.ndarray:
    out = np.zeros(n, dtype=np.float64)
    _check(lib().orc_projected_design_column(C.c_int(k), C.c_int64(n), C.c_int64(ell), _ptr(out)))
    return out


def even_log2_ceil(n: int) -> int:
    out = C.c_int()
    _check(lib().orc_even_log2_ceil(C.c_int64(n), C.byref(out)))
    return out.value


def fwht_unnormalized(v) -> np.ndarray:
    v = np.array(v, copy=True)
    if v.dtype == np.float32:
        _check(lib().orc_fwht_unnormalized_f32(_ptr(v), C.c_size_t(len(v))))
    else:
        v = v.astype(np.float64)
        _check(lib().orc_fwht_unnormalized_f64(_ptr(v), C.c_size_t(len(v))))
    return v


def fwht_normalized(v) -> np.ndarray:
    v = np.array(v, dtype=np.float64, copy=True)
    _check(lib().orc_fwht_normalized_f64(_ptr(v), C.c_size_t(len(v))))
    return v


# --------------------------------------------------------------- sketch ----
class Sketch:
    """sketch.hpp:70-142 — owns the oracle's column-major m x L columns."""

    def __init__(self, handle, a: np.ndarray):
        self._h = C.c_void_p(handle)
        m, n, k, d, L, rn = C.c_int64(), C.c_int64(), C.c_int(), C.c_int64(), C.c_int64(), C.c_double()
        lib().orc_sketch_info(self._h, C.byref(m), C.byref(n), C.byref(k), C.byref(d), C.byref(L), C.byref(rn))
        self.m, self.n, self.k, self.d, self.L = m.value, n.value, k.value, d.value, L.value
        self.row_norm_max = rn.value
        self.dtype = a.dtype
        self.a = a

    def __del__(self):
        if getattr(self, "_h", None) is not None and _lib is not None:
            _lib.orc_sketch_free(self._h)
            self._h = None

    def columns(self) -> np.ndarray:
        """(L, m) view: row ell is column ell of the sketch."""
        ptr = lib().orc_sketch_columns(self._h)
        ct = C.c_double if self.dtype == np.float64 else C.c_float
        buf = (ct * (self.m * self.L)).from_address(ptr)
        buf._owner = self  # keep the sketch alive while any view exists
        return np.ctypeslib.as_array(buf).reshape(self.L, self.m)

    def column(self, ell: int) -> np.ndarray:
        out = np.zeros(self.m, dtype=self.dtype)
        _check(lib().orc_sketch_column(self._h, C.c_int64(ell), _ptr(out)))
        return out


def preprocess(a, dtype=np.float64, threads: int = 1) -> Sketch:
    a = np.ascontiguousarray(a, dtype=dtype)
    if a.ndim != 2:
        raise ValueError("preprocess: A must be 2-D")
    h = C.c_void_p()
    code = 1 if a.dtype == np.float64 else 0
    _check(lib().orc_preprocess(_ptr(a), C.c_int(code), C.c_int64(a.shape[0]), C.c_int64(a.shape[1]),
                                C.c_int(threads), C.byref(h)))
    return Sketch(h.value, a)


def save(sk: Sketch, path: str, with_a: bool = True) -> None:
    """sketch.hpp:215-232 (FSTK v1, fp64)."""
    _check(lib().orc_save(sk._h, str(path).encode(), C.c_int(1 if with_a else 0)))


def load(path: str) -> Sketch:
    """sketch.hpp:241-302."""
    h = C.c_void_p()
    _check(lib().orc_load(str(path).encode(), C.byref(h)))
    sk = Sketch(h.value, np.zeros((0, 0)))
    sk.dtype = np.float64
    return sk


# ------------------------------------------------------------------ rng ----
def rng_u64(seed: int, count: int) -> np.ndarray:
    out = np.zeros(count, dtype=np.uint64)
    lib().orc_rng_u64(C.c_uint64(seed), C.c_int64(count), _ptr(out))
    return out


def rng_index(seed: int, bound: int, count: int) -> np.ndarray:
    out = np.zeros(count, dtype=np.uint64)
    lib().orc_rng_index(C.c_uint64(seed), C.c_uint64(bound), C.c_int64(count), _ptr(out))
    return out


def rng_gaussian(seed: int, count: int) -> np.ndarray:
    out = np.zeros(count, dtype=np.float64)
    lib().orc_rng_gaussian(C.c_uint64(seed), C.c_int64(count), _ptr(out))
    return out


def gen_sparse_targets(seeds, m: int, s: int, value_kind: int = 0, noise_sigma: float = 0.0,
                       threads: int = 0) -> np.ndarray:
    """(B, m) sparse targets, one SeededRng stream per vector (generators.hpp:44-53 draw order,
    +-1/sqrt(s) or N(0,1) values, optional dense N(0, noise_sigma^2) noise)."""
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    Y = np.zeros((len(seeds), m), dtype=np.float64)
    _check(lib().orc_gen_sparse_targets(_ptr(seeds), C.c_int64(len(seeds)), C.c_int64(m), C.c_int64(s),
                                        C.c_int(value_kind), C.c_double(noise_sigma),
                                        C.c_int(threads or (os.cpu_count() or 1)), _ptr(Y)))
    return Y


def rng_unit_double(seed: int, count: int) -> np.ndarray:
    out = np.zeros(count, dtype=np.float64)
    lib().orc_rng_unit_double(C.c_uint64(seed), C.c_int64(count), _ptr(out))
    return out


def rng_coin(seed: int, count: int) -> np.ndarray:
    out = np.zeros(count, dtype=np.uint8)
    lib().orc_rng_coin(C.c_uint64(seed), C.c_int64(count), _ptr(out))
    return out


def mix_seed(z: int) -> int:
    return lib().orc_mix_seed(C.c_uint64(z))


def gen_seed(t: int) -> int:
    return lib().orc_gen_seed(C.c_uint64(t))


def stream_seed(t: int) -> int:
    return lib().orc_stream_seed(C.c_uint64(t))


# --------------------------------------------------------------- stream ----
@dataclass
class StreamParams:
    """stream.hpp:22-39."""
    epsilon: float = 0.0
    delta: float = 0.0
    s: int = 1
    J: int = 1
    K: int = 1
    widen: int = 10
    seed: int = 0

    def validate(self) -> None:
        _check(lib().orc_validate_params(C.c_double(self.epsilon), C.c_double(self.delta), C.c_int64(self.s),
                                         C.c_int64(self.J), C.c_int64(self.K), C.c_int64(self.widen)))


@dataclass
class TransformResult:
    """stream.hpp:41-54."""
    support: np.ndarray
    values: np.ndarray
    candidate_set: np.ndarray
    mu: np.ndarray
    samples_used: int = 0


def choose_params(row_norm_max: float, gamma: float, eta: float, m: int):
    J, K = C.c_int64(), C.c_int64()
    _check(lib().orc_choose_params(C.c_double(row_norm_max), C.c_double(gamma), C.c_double(eta),
                                   C.c_int64(m), C.byref(J), C.byref(K)))
    return J.value, K.value


def candidate_count(s: int, widen: int, m: int) -> int:
    return lib().orc_candidate_count(s, widen, m)


def inner_product_with_design(x, k: int, ell: int) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = C.c_double()
    _check(lib().orc_inner_product_with_design(_ptr(x), C.c_int64(len(x)), C.c_int(k), C.c_int64(ell),
                                               C.byref(out)))
    return out.value


def median_of_batch_means(means: np.ndarray) -> np.ndarray:
    """means: (m, K) -> mu (m)."""
    means = np.asarray(means, dtype=np.float64)
    m, K = means.shape
    colmajor = np.ascontiguousarray(means.T)
    mu = np.zeros(m, dtype=np.float64)
    _check(lib().orc_median_of_batch_means_f64(_ptr(colmajor), C.c_int64(m), C.c_int64(K), _ptr(mu)))
    return mu


def median_of_means(samples: np.ndarray, J: int, K: int) -> np.ndarray:
    """stream.hpp:147-155."""
    samples = np.asarray(samples, dtype=np.float64)
    if J < 1 or K < 1 or samples.shape[1] != J * K:
        raise ValueError("median_of_means: samples must have J*K columns")
    means = np.stack([samples[:, b * J:(b + 1) * J].sum(axis=1) / J for b in range(K)], axis=1)
    return median_of_batch_means(means)


def hard_threshold(v, eps: float) -> np.ndarray:
    """stream.hpp:158-162 — boundary |t| = eps is kept."""
    v = np.asarray(v)
    return np.where(np.abs(v) >= eps, v, 0.0)


def draw_samples(L: int, p: StreamParams) -> np.ndarray:
    out = np.zeros(p.J * p.K if p.J * p.K < (1 << 40) else 0, dtype=np.int64)
    _check(lib().orc_draw_samples(C.c_int64(L), C.c_double(p.epsilon), C.c_double(p.delta), C.c_int64(p.s),
                                  C.c_int64(p.J), C.c_int64(p.K), C.c_int64(p.widen), C.c_uint64(p.seed),
                                  _ptr(out)))
    return out


def transform_with_samples(sk: Sketch, x, p: StreamParams, indices) -> TransformResult:
    return _transform(sk, x, p, np.ascontiguousarray(indices, dtype=np.int64))


def transform(sk: Sketch, x, p: StreamParams) -> TransformResult:
    return _transform(sk, x, p, None)


def _transform(sk: Sketch, x, p: StreamParams, indices) -> TransformResult:
    x = np.ascontiguousarray(x, dtype=sk.dtype)
    if x.shape != (sk.n,):
        raise ValueError("transform: vector length does not match sketch")
    p.validate()
    want = candidate_count(p.s, p.widen, sk.m)
    mu = np.zeros(sk.m, dtype=sk.dtype)
    cand = np.zeros(want, dtype=np.int64)
    sup = np.zeros(want, dtype=np.int64)
    vals = np.zeros(want, dtype=sk.dtype)
    ns = C.c_int64()
    idx_ptr = _ptr(indices) if indices is not None else None
    _check(lib().orc_transform(sk._h, _ptr(x), C.c_double(p.epsilon), C.c_double(p.delta), C.c_int64(p.s),
                               C.c_int64(p.J), C.c_int64(p.K), C.c_int64(p.widen), C.c_uint64(p.seed),
                               idx_ptr, _ptr(mu), _ptr(cand), _ptr(sup), _ptr(vals), C.byref(ns)))
    k = ns.value
    return TransformResult(sup[:k].copy(), vals[:k].copy(), cand, mu, p.J * p.K)


def transform_gathered(a, x, p: StreamParams, indices, gathered, dtype=np.float64) -> TransformResult:
    """draw_and_gather path (stream.hpp:184-191): gathered is (J*K, m), row j = column indices[j].
    dtype float32 runs the same arithmetic in float (Scalar = float)."""
    dtype = np.dtype(dtype)
    a = np.ascontiguousarray(a, dtype=dtype)
    x = np.ascontiguousarray(x, dtype=dtype)
    m, n = a.shape
    indices = np.ascontiguousarray(indices, dtype=np.int64)
    gathered = np.ascontiguousarray(gathered, dtype=dtype)
    if gathered.shape != (p.J * p.K, m):
        raise ValueError("gathered must be (J*K, m)")
    want = candidate_count(p.s, p.widen, m)
    mu = np.zeros(m, dtype=dtype)
    cand = np.zeros(want, dtype=np.int64)
    sup = np.zeros(want, dtype=np.int64)
    vals = np.zeros(want, dtype=dtype)
    ns = C.c_int64()
    fn = lib().orc_transform_gathered if dtype == np.float64 else lib().orc_transform_gathered_f32
    _check(fn(_ptr(a), C.c_int64(m), C.c_int64(n), _ptr(x), C.c_double(p.epsilon),
              C.c_double(p.delta), C.c_int64(p.s), C.c_int64(p.J), C.c_int64(p.K),
              C.c_int64(p.widen), _ptr(indices), _ptr(gathered), _ptr(mu), _ptr(cand),
              _ptr(sup), _ptr(vals), C.byref(ns)))
    k = ns.value
    return TransformResult(sup[:k].copy(), vals[:k].copy(), cand, mu, p.J * p.K)


def transform_gathered_fast_order(a, x, p: StreamParams, indices, gathered) -> TransformResult:
    """The B200 FAST-mode arithmetic restated (lane-partitioned coefficient sums + xor tree, FMA
    accumulation, the refinement's chunked fp64 dot), float32: bit-exact reference for the GPU's
    fp32 FAST path. Same transform as transform_gathered(..., float32) up to summation order."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    x = np.ascontiguousarray(x, dtype=np.float32)
    m, n = a.shape
    indices = np.ascontiguousarray(indices, dtype=np.int64)
    gathered = np.ascontiguousarray(gathered, dtype=np.float32)
    if gathered.shape != (p.J * p.K, m):
        raise ValueError("gathered must be (J*K, m)")
    want = candidate_count(p.s, p.widen, m)
    mu = np.zeros(m, dtype=np.float32)
    cand = np.zeros(want, dtype=np.int64)
    sup = np.zeros(want, dtype=np.int64)
    vals = np.zeros(want, dtype=np.float32)
    ns = C.c_int64()
    _check(lib().orc_transform_gathered_fast_order(_ptr(a), C.c_int64(m), C.c_int64(n), _ptr(x),
                                                   C.c_double(p.epsilon), C.c_double(p.delta), C.c_int64(p.s),
                                                   C.c_int64(p.J), C.c_int64(p.K), C.c_int64(p.widen),
                                                   _ptr(indices), _ptr(gathered), _ptr(mu), _ptr(cand), _ptr(sup),
                                                   _ptr(vals), C.byref(ns)))
    k = ns.value
    return TransformResult(sup[:k].copy(), vals[:k].copy(), cand, mu, p.J * p.K)


def kerdock_block(a, s: int, dtype=np.float64) -> np.ndarray:
    """Kerdock basis s of preprocess(a) (sketch.hpp:171-196): (d, m), row w = column s*d + w."""
    a = np.ascontiguousarray(a, dtype=dtype)
    m, n = a.shape
    d = 1 << even_log2_ceil(n)
    out = np.zeros((d, m), dtype=dtype)
    _check(lib().orc_kerdock_block(_ptr(a), C.c_int(1 if a.dtype == np.float64 else 0), C.c_int64(m),
                                   C.c_int64(n), C.c_int64(s), _ptr(out)))
    return out


def design_columns(k: int, n: int, ells) -> np.ndarray:
    """(count, n): row j = s_{ells[j]} (kerdock.hpp:156-167)."""
    ells = np.ascontiguousarray(ells, dtype=np.int64).ravel()
    out = np.zeros((len(ells), n), dtype=np.float64)
    _check(lib().orc_design_columns(C.c_int(k), C.c_int64(n), _ptr(ells), C.c_int64(len(ells)), _ptr(out)))
    return out


def bench_gathered(a, X, p: StreamParams, seeds, gathered, L: int, threads: int, total: int, predrawn: bool = False):
    """Times the reference transform() over `total` vectors cycling a pool of P prepared vectors.
    gathered: (P, J*K, m) fp64 host columns. Returns (pool support counts, wall seconds)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    X = np.ascontiguousarray(X, dtype=np.float64)
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    gathered = np.ascontiguousarray(gathered, dtype=np.float64)
    m, n = a.shape
    P = X.shape[0]
    counts = np.zeros(P, dtype=np.int64)
    secs = C.c_double()
    _check(lib().orc_bench_gathered(_ptr(a), C.c_int64(m), C.c_int64(n), _ptr(X), C.c_int64(P),
                                    C.c_double(p.epsilon), C.c_double(p.delta), C.c_int64(p.s), C.c_int64(p.J),
                                    C.c_int64(p.K), C.c_int64(p.widen), _ptr(seeds), _ptr(gathered), C.c_int64(L),
                                    C.c_int(threads), C.c_int64(total), _ptr(counts), C.byref(secs),
                                    C.c_int(1 if predrawn else 0)))
    return counts, secs.value


def transform_stream(sk: Sketch, X: np.ndarray, p: StreamParams, seeds: np.ndarray, threads: int):
    """Runs transform() over B vectors on `threads` host threads; returns (counts, seconds)."""
    X = np.ascontiguousarray(X, dtype=sk.dtype)
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    B = X.shape[0]
    counts = np.zeros(B, dtype=np.int64)
    secs = C.c_double()
    _check(lib().orc_transform_stream(sk._h, _ptr(X), C.c_int64(B), C.c_double(p.epsilon), C.c_double(p.delta),
                                      C.c_int64(p.s), C.c_int64(p.J), C.c_int64(p.K), C.c_int64(p.widen),
                                      _ptr(seeds), C.c_int(threads), _ptr(counts), C.byref(secs)))
    return counts, secs.value


# ----------------------------------------------------------- generators ----
def gen_orthogonal(n: int, seed: int) -> np.ndarray:
    out = np.zeros((n, n), dtype=np.float64)
    _check(lib().orc_gen_orthogonal(C.c_int64(n), C.c_uint64(seed), _ptr(out)))
    return out


def gen_mixture(a: np.ndarray, p: float, seed: int):
    """generators.hpp:60-85 -> (x, truth), both rescaled by |A^T y|."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    m, n = a.shape
    x = np.zeros(n)
    truth = np.zeros(m)
    _check(lib().orc_gen_mixture(_ptr(a), C.c_int64(m), C.c_int64(n), C.c_double(p), C.c_uint64(seed), _ptr(x),
                                 _ptr(truth)))
    return x, truth


def gen_exact_sparse(a: np.ndarray, s: int, seed: int):
    a = np.ascontiguousarray(a, dtype=np.float64)
    m, n = a.shape
    x = np.zeros(n, dtype=np.float64)
    truth = np.zeros(m, dtype=np.float64)
    _check(lib().orc_gen_exact_sparse(_ptr(a), C.c_int64(m), C.c_int64(n), C.c_int64(s), C.c_uint64(seed),
                                      _ptr(x), _ptr(truth)))
    return x, truth


# ---- design verifiers (kerdock.hpp:198-317, cli.hpp:45-60) ----
class MubReport(NamedTuple):
    max_within_gram_dev: float
    min_cross_sq: float
    max_cross_sq: float
    max_cross_dev: float
    exhaustive: bool

    def passed(self, tol: float) -> bool:
        return self.max_within_gram_dev <= tol and self.max_cross_dev <= tol


class MomentReport(NamedTuple):
    m1: float
    m2: float
    exact: bool


def materialize_design(k: int) -> np.ndarray:
    """(L, d): row c = unit design vector u_c (the reference's d x L columns)."""
    d = 1 << k
    L = d * (d // 2 + 1)
    out = np.zeros((L, d), dtype=np.float64)
    _check(lib().orc_materialize_design(C.c_int(k), _ptr(out)))
    return out


def verify_mub(k: int, cap: int = 8) -> MubReport:
    out = np.zeros(4)
    ex = C.c_int()
    _check(lib().orc_verify_mub(C.c_int(k), C.c_int(cap), _ptr(out), C.byref(ex)))
    return MubReport(*[float(v) for v in out], bool(ex.value))


def verify_design_moments(k: int, cap: int = 8) -> MomentReport:
    out = np.zeros(2)
    ex = C.c_int()
    _check(lib().orc_verify_design_moments(C.c_int(k), C.c_int(cap), _ptr(out), C.byref(ex)))
    return MomentReport(float(out[0]), float(out[1]), bool(ex.value))


def design_moments_of(u) -> MomentReport:
    """u: (L, d) rows = columns of the reference's d x L matrix."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.zeros(2)
    _check(lib().orc_design_moments_of(_ptr(u), C.c_int64(u.shape[1]), C.c_int64(u.shape[0]), _ptr(out)))
    return MomentReport(float(out[0]), float(out[1]), True)


def design_moment_target(d: int, k: int) -> float:
    return float(lib().orc_design_moment_target(C.c_int64(d), C.c_int(k)))


def verify_kerdock_set(k: int):
    """(skew-symmetric with zero diagonal, rank-deficient pair count)."""
    skew = C.c_int()
    bad = C.c_int64()
    _check(lib().orc_verify_kerdock_set(C.c_int(k), C.byref(skew), C.byref(bad)))
    return bool(skew.value), int(bad.value)


def bench_preprocess(a, bases: int, threads: int) -> float:
    """Wall seconds of the reference per-basis preprocessing for the first `bases` Kerdock bases."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    secs = C.c_double()
    _check(lib().orc_bench_preprocess(_ptr(a), C.c_int64(a.shape[0]), C.c_int64(a.shape[1]), C.c_int64(bases),
                                      C.c_int(threads), C.byref(secs)))
    return secs.value
