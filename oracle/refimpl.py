"""ORACLE / TEST INFRASTRUCTURE ONLY.

ctypes front-end over ``oracle/_ref/libfst_ref.so``: the REFERENCE's own hot-path
code (proj/include/fst/sketch.hpp, stream.hpp, kerdock.hpp, ...) compiled unmodified
from /root/reference against the Eigen-API shim in ``oracle/eigen_shim`` (see
``oracle/ref_capi.cpp``). ``make -C oracle ref`` builds it where /root/reference
exists; the built .so travels with the repo snapshot. Only ``tests/`` and
``bench.py``'s CPU legs use this module.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import oracle as orc

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libfst_ref.so")
_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} not built (make -C oracle ref, needs /root/reference)")
        _lib = C.CDLL(LIB_PATH)
        _lib.fstref_last_error.restype = C.c_char_p
        _lib.fstref_sketch_free.argtypes = [C.c_void_p]
    return _lib


def _check(rc: int) -> None:
    if rc != 0:
        raise orc._ERRORS.get(rc, RuntimeError)(lib().fstref_last_error().decode())


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class RefSketch:
    """fst::Sketch built by the reference's preprocess() (or without columns)."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle)
        m, n, L, rn = C.c_int64(), C.c_int64(), C.c_int64(), C.c_double()
        _check(lib().fstref_sketch_info(self._h, C.byref(m), C.byref(n), C.byref(L), C.byref(rn)))
        self.m, self.n, self.L, self.row_norm_max = m.value, n.value, L.value, rn.value

    def __del__(self):
        if getattr(self, "_h", None) is not None and _lib is not None:
            _lib.fstref_sketch_free(self._h)
            self._h = None

    def columns(self) -> np.ndarray:
        """(L, m): row ell = column A s_ell."""
        out = np.zeros((self.L, self.m), dtype=np.float64)
        _check(lib().fstref_sketch_columns(self._h, _ptr(out)))
        return out


def preprocess(a, threads: int = 1) -> RefSketch:
    a = np.ascontiguousarray(a, dtype=np.float64)
    h = C.c_void_p()
    _check(lib().fstref_preprocess(_ptr(a), C.c_int64(a.shape[0]), C.c_int64(a.shape[1]), C.c_int(threads),
                                   C.byref(h)))
    return RefSketch(h.value)


def sketch_without_columns(a) -> RefSketch:
    a = np.ascontiguousarray(a, dtype=np.float64)
    h = C.c_void_p()
    _check(lib().fstref_sketch_without_columns(_ptr(a), C.c_int64(a.shape[0]), C.c_int64(a.shape[1]),
                                               C.byref(h)))
    return RefSketch(h.value)


def draw_samples(sk: RefSketch, p) -> np.ndarray:
    out = np.zeros(p.J * p.K, dtype=np.int64)
    _check(lib().fstref_draw_samples(sk._h, C.c_double(p.epsilon), C.c_double(p.delta), C.c_int64(p.s),
                                     C.c_int64(p.J), C.c_int64(p.K), C.c_int64(p.widen), C.c_uint64(p.seed),
                                     _ptr(out)))
    return out


def transform(sk: RefSketch, x, p, gathered=None) -> "orc.TransformResult":
    """fst::transform; gathered (N, m) switches to the draw_and_gather form."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    want = orc.candidate_count(p.s, p.widen, sk.m)
    mu = np.zeros(sk.m)
    cand = np.zeros(want, dtype=np.int64)
    sup = np.zeros(want, dtype=np.int64)
    vals = np.zeros(want)
    ns = C.c_int64()
    g = None if gathered is None else np.ascontiguousarray(gathered, dtype=np.float64)
    _check(lib().fstref_transform(sk._h, _ptr(x), C.c_int64(x.shape[0]), C.c_double(p.epsilon), C.c_double(p.delta), C.c_int64(p.s),
                                  C.c_int64(p.J), C.c_int64(p.K), C.c_int64(p.widen), C.c_uint64(p.seed), _ptr(g),
                                  _ptr(mu), _ptr(cand), _ptr(sup), _ptr(vals), C.byref(ns)))
    k = ns.value
    return orc.TransformResult(sup[:k].copy(), vals[:k].copy(), cand, mu, p.J * p.K)


def choose_params(row_norm_max: float, gamma: float, eta: float, m: int):
    J, K = C.c_int64(), C.c_int64()
    _check(lib().fstref_choose_params(C.c_double(row_norm_max), C.c_double(gamma), C.c_double(eta), C.c_int64(m),
                                      C.byref(J), C.byref(K)))
    return J.value, K.value


def bench_gathered(a, X, p, seeds, gathered, threads: int, total: int):
    """The reference's draw_samples + transform_with_samples over `total` vectors cycling the P
    prepared vectors (gathered: (P, J*K, m) fp64 columns). Returns (pool support counts, seconds)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    X = np.ascontiguousarray(X, dtype=np.float64)
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    gathered = np.ascontiguousarray(gathered, dtype=np.float64)
    m, n = a.shape
    P = X.shape[0]
    counts = np.zeros(P, dtype=np.int64)
    secs = C.c_double()
    _check(lib().fstref_bench_gathered(_ptr(a), C.c_int64(m), C.c_int64(n), _ptr(X), C.c_int64(P),
                                       C.c_double(p.epsilon), C.c_double(p.delta), C.c_int64(p.s), C.c_int64(p.J),
                                       C.c_int64(p.K), C.c_int64(p.widen), _ptr(seeds), _ptr(gathered),
                                       C.c_int(threads), C.c_int64(total), _ptr(counts), C.byref(secs)))
    return counts, secs.value
