"""Python mirror of the reference ``fst`` API for the thresholded-Ax hot path.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/fst/{sketch,stream}.hpp — ``preprocess``,
``Sketch``, ``StreamParams``, ``choose_params``, ``draw_samples``,
``transform``, ``transform_with_samples``, ``TransformResult`` — plus the
batched stream entry point ``transform_batch`` the GPU is built around. Every
call goes through the C-ABI in ``include/fst_b200.h`` (libfst_b200.so, sm_100a
kernels). There is no CPU fallback: without the built library or a B200 the
calls raise.

Exception mapping (reference -> Python): std::invalid_argument -> ValueError,
std::out_of_range -> IndexError, std::overflow_error -> OverflowError,
std::runtime_error (allocation) -> MemoryError, CUDA failure -> CudaError,
unsupported shape -> NotSupportedError.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfst_b200.so")

F32, F64 = 0, 1
MODE_DEFAULT, MODE_FAST, MODE_STRICT = 0, 1, 2


class CudaError(RuntimeError):
    """CUDA runtime failure or no sm_100 device (no CPU fallback exists)."""


class NotSupportedError(RuntimeError):
    """Shape outside this build's GPU limits."""


class IoError(OSError):
    """io.hpp:23 IoError."""


class MagicMismatchError(IoError):
    """io.hpp:26"""


class VersionUnsupportedError(IoError):
    """io.hpp:29"""


class TruncatedPayloadError(IoError):
    """io.hpp:32"""


class MalformedHeaderError(IoError):
    """io.hpp:35"""


class NoMatrixError(RuntimeError):
    """sketch.hpp:109 logic_error: the sketch has no embedded matrix."""


_ERRORS = {1: ValueError, 2: IndexError, 3: OverflowError, 4: MemoryError, 5: CudaError, 6: NotSupportedError,
           7: IoError, 8: MagicMismatchError, 9: VersionUnsupportedError, 10: TruncatedPayloadError,
           11: MalformedHeaderError, 12: NoMatrixError}


class _Params(C.Structure):
    _fields_ = [("epsilon", C.c_double), ("delta", C.c_double), ("s", C.c_int64), ("J", C.c_int64),
                ("K", C.c_int64), ("widen", C.c_int64), ("seed", C.c_uint64), ("mode", C.c_int32),
                ("reserved", C.c_int32)]


class _Info(C.Structure):
    _fields_ = [("m", C.c_int64), ("n", C.c_int64), ("d", C.c_int64), ("L", C.c_int64), ("k", C.c_int32),
                ("dtype", C.c_int32), ("row_norm_max", C.c_double), ("device", C.c_int32),
                ("reserved", C.c_int32), ("column_stride", C.c_int64), ("device_bytes", C.c_uint64),
                ("preprocess_ms", C.c_double)]


_lib = None

# Every symbol the C-ABI header declares (checked by tests/test_abi.py).
EXPORTED = [
    "fstg_last_error", "fstg_version", "fstg_device_count", "fstg_even_log2_ceil", "fstg_design_params",
    "fstg_kerdock_matrix", "fstg_choose_params", "fstg_validate_params", "fstg_candidate_count",
    "fstg_preprocess", "fstg_preprocess_shard", "fstg_sketch_info_get", "fstg_row_norm_max",
    "fstg_sketch_column", "fstg_sketch_gather", "fstg_sketch_device_columns", "fstg_sketch_preprocess_ms", "fstg_destroy",
    "fstg_draw_samples", "fstg_transform_batch", "fstg_transform_with_samples_batch", "fstg_profile_enable",
    "fstg_profile_reset", "fstg_profile_read", "fstg_launch_count", "fstg_set_pool_retain", "fstg_gen_gaussian",
    "fstg_gen_sparse_targets", "fstg_save", "fstg_load", "fstg_gen_mixture_targets",
    "fstg_preprocess_design", "fstg_sample_columns", "fstg_transform_gathered_batch",
    "fstg_verify_mub", "fstg_verify_design_moments", "fstg_design_moment_target", "fstg_verify_kerdock_set",
    "fstg_transform_design_batch", "fstg_design_partial_means", "fstg_transform_from_means",
    "fstg_inner_product_with_design", "fstg_median_of_means", "fstg_hard_threshold", "fstg_projected_design_column",
    "fstg_sketch_embedded_matrix",
]


def lib():
    """Loads libfst_b200.so (raises if it was not built — no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (make -C "
                              f"paper_2105_05879_b200/csrc)")
        L = C.CDLL(LIB_PATH)
        L.fstg_last_error.restype = C.c_char_p
        L.fstg_version.restype = C.c_char_p
        L.fstg_candidate_count.restype = C.c_int64
        L.fstg_candidate_count.argtypes = [C.c_int64, C.c_int64, C.c_int64]
        L.fstg_destroy.argtypes = [C.c_void_p]
        L.fstg_destroy.restype = None
        L.fstg_design_moment_target.restype = C.c_double
        L.fstg_design_moment_target.argtypes = [C.c_int64, C.c_int]
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc != 0:
        raise _ERRORS.get(rc, RuntimeError)(lib().fstg_last_error().decode())


def device_count() -> int:
    c = C.c_int()
    _check(lib().fstg_device_count(C.byref(c)))
    return c.value


# -------------------------------------------------------------- pointers ----
def _is_torch(t) -> bool:
    return type(t).__module__.startswith("torch")


def _ptr(a) -> C.c_void_p:
    if a is None:
        return C.c_void_p(None)
    if _is_torch(a):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return C.c_void_p(a.data_ptr())
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return C.c_void_p(a.ctypes.data)
    raise TypeError(f"unsupported buffer type {type(a)}")


def _dtype_code(dt) -> int:
    s = str(dt)
    if "float64" in s or s == "double":
        return F64
    if "float32" in s or s == "float":
        return F32
    raise ValueError(f"dtype must be float32 or float64, got {dt}")


# ----------------------------------------------------------- host helpers ----
def even_log2_ceil(n: int) -> int:
    """sketch.hpp:58-63"""
    k = C.c_int()
    _check(lib().fstg_even_log2_ceil(C.c_int64(n), C.byref(k)))
    return k.value


def design_params(k: int):
    """kerdock.hpp:26-31 -> (d, L)"""
    d, L = C.c_int64(), C.c_int64()
    _check(lib().fstg_design_params(C.c_int(k), C.byref(d), C.byref(L)))
    return d.value, L.value


def kerdock_matrix(k: int, s: int) -> np.ndarray:
    """kerdock.hpp:55-84 (bit j of row i = entry (i, j))"""
    out = np.zeros(k, dtype=np.uint64)
    _check(lib().fstg_kerdock_matrix(C.c_int(k), C.c_uint64(s), out.ctypes.data_as(C.c_void_p)))
    return out


def choose_params(row_norm_max: float, gamma: float, eta: float, m: int):
    """stream.hpp:58-69 -> (J, K)"""
    J, K = C.c_int64(), C.c_int64()
    _check(lib().fstg_choose_params(C.c_double(row_norm_max), C.c_double(gamma), C.c_double(eta), C.c_int64(m),
                                    C.byref(J), C.byref(K)))
    return J.value, K.value


def candidate_count(s: int, widen: int, m: int) -> int:
    """stream.hpp:245-246 (`want`)"""
    return int(lib().fstg_candidate_count(s, widen, m))


@dataclass
class StreamParams:
    """stream.hpp:22-39; ``mode`` selects FAST (fp32 default) or STRICT (fp64 default) arithmetic."""
    epsilon: float = 0.0
    delta: float = 0.0
    s: int = 1
    J: int = 1
    K: int = 1
    widen: int = 10
    seed: int = 0
    mode: int = MODE_DEFAULT

    def _c(self) -> _Params:
        return _Params(self.epsilon, self.delta, self.s, self.J, self.K, self.widen, self.seed & (2**64 - 1),
                       self.mode, 0)

    def validate(self) -> None:
        p = self._c()
        _check(lib().fstg_validate_params(C.byref(p)))


@dataclass
class TransformResult:
    """stream.hpp:41-54: sorted support with exact values, the candidate set and mu."""
    support: np.ndarray
    values: np.ndarray
    candidate_set: np.ndarray
    mu: np.ndarray
    samples_used: int


@dataclass
class BatchResult:
    """Batched outputs (row v belongs to vector v; first counts[v] support entries valid)."""
    counts: object
    support: object
    values: object
    candidates: object = None
    mu: object = None

    def result(self, v: int, samples_used: int = 0) -> TransformResult:
        c = int(_to_numpy(self.counts)[v])
        sup = _to_numpy(self.support)[v, :c].astype(np.int64)
        val = _to_numpy(self.values)[v, :c].copy()
        cand = _to_numpy(self.candidates)[v].astype(np.int64) if self.candidates is not None else None
        mu = _to_numpy(self.mu)[v].copy() if self.mu is not None else None
        return TransformResult(sup, val, cand, mu, samples_used)


def _to_numpy(a):
    if a is None:
        return None
    if _is_torch(a):
        return a.detach().cpu().numpy()
    return a


# ----------------------------------------------------------------- sketch ----
class Sketch:
    """sketch.hpp:70-142 — device-resident {A s_l} (column-major m x L) + embedded A."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        info = _Info()
        _check(lib().fstg_sketch_info_get(self._h, C.byref(info)))
        self.m, self.n, self.d, self.L, self.k = info.m, info.n, info.d, info.L, info.k
        self.dtype = np.float64 if info.dtype == F64 else np.float32
        self.device = info.device
        self.column_stride = info.column_stride
        self.device_bytes = info.device_bytes
        self.preprocess_ms = info.preprocess_ms
        self._row_norm_max = info.row_norm_max

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().fstg_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self):
        return self._h

    def row_norm_max(self) -> float:
        return self._row_norm_max

    def kerdock_bases(self) -> int:
        return self.d // 2

    def column(self, ell: int) -> np.ndarray:
        """Sketch::column (sketch.hpp:114-117), copied to host."""
        out = np.zeros(self.m, dtype=self.dtype)
        _check(lib().fstg_sketch_column(self._h, C.c_int64(ell), out.ctypes.data_as(C.c_void_p)))
        return out

    def embedded_matrix(self) -> np.ndarray:
        """Sketch::embedded_matrix (sketch.hpp:107-111): A (m, n), copied to host."""
        out = np.zeros((self.m, self.n), dtype=self.dtype)
        _check(lib().fstg_sketch_embedded_matrix(self._h, _ptr(out)))
        return out

    def gather(self, indices) -> np.ndarray:
        """draw_and_gather (stream.hpp:184-191): (count, m) host array of columns indices[j]."""
        idx = np.ascontiguousarray(indices, dtype=np.int64).ravel()
        out = np.zeros((len(idx), self.m), dtype=self.dtype)
        _check(lib().fstg_sketch_gather(self._h, _ptr(idx), C.c_int64(len(idx)), _ptr(out), C.c_void_p(None)))
        return out

    def device_columns_ptr(self) -> int:
        p = C.c_void_p()
        _check(lib().fstg_sketch_device_columns(self._h, C.byref(p)))
        return p.value


def preprocess(a, device: int = 0, stream: Optional[int] = None) -> Sketch:
    """sketch.hpp:149-211. ``a``: m x n float32/float64, numpy (host) or torch (host/cuda)."""
    if _is_torch(a):
        a = a.contiguous()
        dt, shape = a.dtype, tuple(a.shape)
    else:
        a = np.ascontiguousarray(a)
        if a.dtype not in (np.float32, np.float64):
            a = a.astype(np.float64)
        dt, shape = a.dtype, a.shape
    if len(shape) != 2:
        raise ValueError("preprocess: matrix must be 2-D")
    m, n = shape
    if m < 1 or n < 1:
        raise ValueError("preprocess: matrix must be nonempty")
    h = C.c_void_p()
    _check(lib().fstg_preprocess(_ptr(a), C.c_int(_dtype_code(dt)), C.c_int64(m), C.c_int64(n), C.c_int(device),
                                 C.c_void_p(stream), C.byref(h)))
    return Sketch(h.value)


def preprocess_design(a, device: int = 0, stream: Optional[int] = None) -> Sketch:
    """Design-only sketch (embedded A + Kerdock tables, no columns) for n whose sketch cannot exist."""
    a = a.contiguous() if _is_torch(a) else np.ascontiguousarray(a)
    m, n = tuple(a.shape)
    h = C.c_void_p()
    _check(lib().fstg_preprocess_design(_ptr(a), C.c_int(_dtype_code(a.dtype)), C.c_int64(m), C.c_int64(n),
                                        C.c_int(device), C.c_void_p(stream), C.byref(h)))
    return Sketch(h.value)


def sample_columns(sk: Sketch, indices, out=None, stream: Optional[int] = None):
    """Retain-sampled preprocessing: columns A s_ell for the given indices, (count, column_stride)."""
    if not _is_torch(indices):
        indices = np.ascontiguousarray(indices, dtype=np.int64).ravel()
    count = int(indices.numel() if _is_torch(indices) else indices.size)
    if out is None:
        out = np.zeros((count, sk.column_stride), dtype=sk.dtype)
    _check(lib().fstg_sample_columns(sk.handle, _ptr(indices), C.c_int64(count), _ptr(out), C.c_void_p(stream)))
    return out


def transform_gathered_batch(sk: Sketch, X, p: StreamParams, indices, gathered, *, candidates: bool = False,
                             mu: bool = False, out: Optional[BatchResult] = None,
                             stream: Optional[int] = None) -> BatchResult:
    """transform_with_samples with drawn.use_gathered (stream.hpp:235-236): columns from `gathered`
    (device tensor, B*J*K x column_stride), indices (B x J*K) for the coefficients."""
    X = _prep_x(sk, X)
    B = X.shape[0]
    p.validate()
    want = candidate_count(p.s, p.widen, sk.m)
    if out is None:
        out = _alloc_outputs(_is_torch(X) and X.is_cuda, B, want, sk.m, sk.dtype, candidates, mu, sk.device)
    else:
        _check_outputs(out, B, want, sk.m, sk.dtype, None)
    _check_buf("indices", indices, (B, p.J * p.K), ("int64",))
    pc = p._c()
    _check(lib().fstg_transform_gathered_batch(sk.handle, _ptr(X), C.c_int64(B), C.byref(pc), _ptr(indices),
                                               _ptr(gathered), _ptr(out.counts), _ptr(out.support), _ptr(out.values),
                                               _ptr(out.candidates), _ptr(out.mu), C.c_void_p(stream)))
    return out


def preprocess_shard(a, basis_begin: int, basis_end: int, include_identity: bool, device: int = 0,
                     stream: Optional[int] = None) -> Sketch:
    """Basis-sharded build of a full-size sketch (only bases [begin, end) computed)."""
    a = a.contiguous() if _is_torch(a) else np.ascontiguousarray(a)
    m, n = tuple(a.shape)
    h = C.c_void_p()
    _check(lib().fstg_preprocess_shard(_ptr(a), C.c_int(_dtype_code(a.dtype)), C.c_int64(m), C.c_int64(n),
                                       C.c_int(device), C.c_void_p(stream), C.c_int64(basis_begin),
                                       C.c_int64(basis_end), C.c_int(1 if include_identity else 0), C.byref(h)))
    return Sketch(h.value)


def transform_design_batch(sk: Sketch, X, p: StreamParams, seeds=None, *, row_block: int = 0,
                           candidates: bool = False, mu: bool = False, out: Optional[BatchResult] = None,
                           stream: Optional[int] = None) -> BatchResult:
    """transform (stream.hpp:272-275) for a batch on a design-only sketch (no columns exist):
    row blocks of the sampled columns are computed and consumed in turn (one Kerdock pass per call).
    X, seeds and outputs are device tensors."""
    import torch
    X = _prep_x(sk, X)
    if not (_is_torch(X) and X.is_cuda):
        raise ValueError("transform_design_batch: X must be a CUDA tensor")
    B = X.shape[0]
    p.validate()
    want = candidate_count(p.s, p.widen, sk.m)
    if out is None:
        out = _alloc_outputs(True, B, want, sk.m, sk.dtype, candidates, mu, sk.device)
    else:
        _check_outputs(out, B, want, sk.m, sk.dtype, _buf_info(X)[2])
    if seeds is not None and not (_is_torch(seeds) and seeds.is_cuda):
        seeds = torch.from_numpy(np.ascontiguousarray(seeds, dtype=np.uint64).view(np.int64)).to(X.device)
    _check_seeds(seeds, B)
    pc = p._c()
    _check(lib().fstg_transform_design_batch(sk.handle, _ptr(X), C.c_int64(B), C.byref(pc), _ptr(seeds),
                                             C.c_int64(row_block), _ptr(out.counts), _ptr(out.support),
                                             _ptr(out.values), _ptr(out.candidates), _ptr(out.mu),
                                             C.c_void_p(stream)))
    return out


def _dev_seeds(seeds, device):
    import torch
    if seeds is None or (_is_torch(seeds) and seeds.is_cuda):
        return seeds
    return torch.from_numpy(np.ascontiguousarray(seeds, dtype=np.uint64).view(np.int64)).to(device)


def design_partial_means(sk: Sketch, X, p: StreamParams, seeds=None, row_begin: int = 0, row_end: Optional[int] = None,
                         *, row_block: int = 0, out=None, stream: Optional[int] = None):
    """Rows [row_begin, row_end) of every vector's K batch means on a design-only sketch:
    a (B, K, row_end - row_begin) device tensor (one Kerdock pass over those rows)."""
    import torch
    X = _prep_x(sk, X)
    if not (_is_torch(X) and X.is_cuda):
        raise ValueError("design_partial_means: X must be a CUDA tensor")
    p.validate()
    row_end = sk.m if row_end is None else row_end
    B, h = X.shape[0], row_end - row_begin
    if out is None:
        out = torch.empty((B, p.K, h), dtype=X.dtype, device=X.device)
    elif (out.dim() != 3 or tuple(out.shape[:2]) != (B, p.K) or out.shape[2] < h or out.dtype != X.dtype
          or out.device != X.device or out.stride(2) != 1):
        raise ValueError("design_partial_means: out must be a (B, K, >= rows) tensor like X")
    seeds = _dev_seeds(seeds, X.device)
    _check_seeds(seeds, B)
    _check(lib().fstg_design_partial_means(sk.handle, _ptr(X), C.c_int64(B), C.byref(p._c()), _ptr(seeds),
                                           C.c_int64(row_begin), C.c_int64(row_end), C.c_int64(row_block), _ptr(out),
                                           C.c_int64(out.stride(0)), C.c_int64(out.stride(1)), C.c_void_p(stream)))
    return out


def transform_from_means(sk: Sketch, X, p: StreamParams, means, *, candidates: bool = False, mu: bool = False,
                         out: Optional[BatchResult] = None, stream: Optional[int] = None) -> BatchResult:
    """Median / top-want / refinement from complete batch means: means is a (B, K + 1, ld)
    device tensor (ld >= m, 16-byte multiple; slot K is overwritten with mu)."""
    X = _prep_x(sk, X)
    if not (_is_torch(X) and X.is_cuda):
        raise ValueError("transform_from_means: X must be a CUDA tensor")
    p.validate()
    B = X.shape[0]
    want = candidate_count(p.s, p.widen, sk.m)
    if out is None:
        out = _alloc_outputs(True, B, want, sk.m, sk.dtype, candidates, mu, sk.device)
    else:
        _check_outputs(out, B, want, sk.m, sk.dtype, _buf_info(X)[2])
    if means.dim() != 3 or means.shape[0] != B or means.shape[1] < p.K + 1 or means.shape[2] < sk.m:
        raise ValueError("transform_from_means: means must be (B, K + 1, ld >= m)")
    _check(lib().fstg_transform_from_means(sk.handle, _ptr(X), C.c_int64(B), C.byref(p._c()), _ptr(means),
                                           C.c_int64(means.stride(0)), C.c_int64(means.stride(1)), _ptr(out.counts),
                                           _ptr(out.support), _ptr(out.values), _ptr(out.candidates), _ptr(out.mu),
                                           C.c_void_p(stream)))
    return out


def save(sk: Sketch, path, version: int = 1) -> None:
    """sketch.hpp:215-232: FSTK v1 (float64, the reference's format) or v2 (float32)."""
    _check(lib().fstg_save(sk.handle, str(path).encode(), C.c_int(version)))


def load(path, dtype=None, device: int = 0, stream: Optional[int] = None) -> Sketch:
    """sketch.hpp:241-302 straight into HBM. dtype None: keep the file's precision."""
    if dtype is None:
        try:
            with open(path, "rb") as f:
                head = f.read(8)
        except OSError:
            head = b""  # the library reports the IoError
        dtype = np.float32 if len(head) == 8 and head[:4] == b"FSTK" and head[4] == 2 else np.float64
    h = C.c_void_p()
    _check(lib().fstg_load(str(path).encode(), C.c_int(_dtype_code(np.dtype(dtype))), C.c_int(device),
                           C.c_void_p(stream), C.byref(h)))
    return Sketch(h.value)


# ----------------------------------------------------------------- stream ----
def draw_samples(sk: Sketch, p: StreamParams, seeds=None, B: Optional[int] = None) -> np.ndarray:
    """stream.hpp:173-182 on the GPU. Returns (J*K,) or, with per-vector seeds, (B, J*K) int64."""
    p.validate()
    N = p.J * p.K
    if seeds is None:
        out = np.zeros((1 if B is None else B, N), dtype=np.int64)
        sp = None
    else:
        seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
        out = np.zeros((len(seeds), N), dtype=np.int64)
        sp = seeds
    pc = p._c()
    _check(lib().fstg_draw_samples(sk.handle, C.byref(pc), _ptr(sp), C.c_int64(out.shape[0]), _ptr(out),
                                   C.c_void_p(None)))
    return out[0] if (seeds is None and B is None) else out


def _alloc_outputs(like_torch, B, want, m, dtype, want_cands, want_mu, device):
    if like_torch:
        import torch
        tdt = torch.float64 if dtype == np.float64 else torch.float32
        dev = f"cuda:{device}"
        return BatchResult(torch.zeros(B, dtype=torch.int32, device=dev),
                           torch.zeros((B, want), dtype=torch.int32, device=dev),
                           torch.zeros((B, want), dtype=tdt, device=dev),
                           torch.zeros((B, want), dtype=torch.int32, device=dev) if want_cands else None,
                           torch.zeros((B, m), dtype=tdt, device=dev) if want_mu else None)
    return BatchResult(np.zeros(B, dtype=np.int32), np.zeros((B, want), dtype=np.int32),
                       np.zeros((B, want), dtype=dtype),
                       np.zeros((B, want), dtype=np.int32) if want_cands else None,
                       np.zeros((B, m), dtype=dtype) if want_mu else None)


def _buf_info(a):
    """(shape, dtype name, device tag) of a numpy array or torch tensor."""
    if _is_torch(a):
        return tuple(a.shape), str(a.dtype).split(".")[-1], ("cuda:%d" % a.device.index if a.is_cuda else "cpu")
    a = np.asarray(a)
    return a.shape, a.dtype.name, "cpu"


def _check_buf(name, a, shape, dtypes, device=None):
    """Rejects a caller buffer the C-ABI would read or write past (wrong length / dtype / device)."""
    if a is None:
        return
    shp, dt, dev = _buf_info(a)
    if tuple(shp) != tuple(shape):
        raise ValueError(f"{name}: shape {tuple(shp)} != {tuple(shape)}")
    if dt not in dtypes:
        raise ValueError(f"{name}: dtype {dt} not in {dtypes}")
    if device is not None and dev != device:
        raise ValueError(f"{name}: on {dev}, expected {device}")


def _check_seeds(seeds, B):
    if seeds is not None:
        _check_buf("seeds", seeds, (B,), ("int64", "uint64"))


def _check_outputs(out: "BatchResult", B, want, m, dtype, like):
    """Every output buffer must hold B vectors of the right width and dtype, all on the same side
    (host or the sketch's device) as `like` decides."""
    vdt = np.dtype(dtype).name
    dev = _buf_info(out.counts)[2]
    if like is not None and like != dev:
        raise ValueError(f"outputs on {dev} but inputs on {like}")
    _check_buf("counts", out.counts, (B,), ("int32",), dev)
    _check_buf("support", out.support, (B, want), ("int32",), dev)
    _check_buf("values", out.values, (B, want), (vdt,), dev)
    _check_buf("candidates", out.candidates, (B, want), ("int32",), dev)
    _check_buf("mu", out.mu, (B, m), (vdt,), dev)


def _prep_x(sk: Sketch, X):
    if _is_torch(X):
        X = X.contiguous()
    else:
        X = np.ascontiguousarray(X, dtype=sk.dtype)
    if str(X.dtype).split(".")[-1] != np.dtype(sk.dtype).name:
        raise ValueError("transform: vector dtype does not match sketch")
    if X.ndim == 1:
        X = X.reshape(1, -1)
    if X.shape[1] != sk.n:
        raise ValueError("transform: vector length does not match sketch")
    return X


def transform_batch(sk: Sketch, X, p: StreamParams, seeds=None, *, candidates: bool = False, mu: bool = False,
                    out: Optional[BatchResult] = None, stream: Optional[int] = None) -> BatchResult:
    """transform (stream.hpp:272-275) over a batch X (B x n). seeds: per-vector seeds (None -> p.seed)."""
    X = _prep_x(sk, X)
    B = X.shape[0]
    want = candidate_count(p.s, p.widen, sk.m)
    p.validate()
    if out is None:
        out = _alloc_outputs(_is_torch(X) and X.is_cuda, B, want, sk.m, sk.dtype, candidates, mu, sk.device)
    else:
        _check_outputs(out, B, want, sk.m, sk.dtype, None)
    if seeds is not None and not _is_torch(seeds):
        seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    _check_seeds(seeds, B)
    pc = p._c()
    _check(lib().fstg_transform_batch(sk.handle, _ptr(X), C.c_int64(B), C.byref(pc), _ptr(seeds),
                                      _ptr(out.counts), _ptr(out.support), _ptr(out.values),
                                      _ptr(out.candidates), _ptr(out.mu), C.c_void_p(stream)))
    return out


def transform_with_samples_batch(sk: Sketch, X, p: StreamParams, indices, *, candidates: bool = False,
                                 mu: bool = False, out: Optional[BatchResult] = None,
                                 stream: Optional[int] = None) -> BatchResult:
    """transform_with_samples (stream.hpp:197-268) with pre-drawn indices (B x J*K int64)."""
    X = _prep_x(sk, X)
    B = X.shape[0]
    p.validate()
    if not _is_torch(indices):
        indices = np.ascontiguousarray(indices, dtype=np.int64).reshape(B, -1)
    if tuple(indices.shape) != (B, p.J * p.K):
        raise ValueError("transform: drawn sample count does not match J*K")
    _check_buf("indices", indices, (B, p.J * p.K), ("int64",))
    want = candidate_count(p.s, p.widen, sk.m)
    if out is None:
        out = _alloc_outputs(_is_torch(X) and X.is_cuda, B, want, sk.m, sk.dtype, candidates, mu, sk.device)
    else:
        _check_outputs(out, B, want, sk.m, sk.dtype, None)
    pc = p._c()
    _check(lib().fstg_transform_with_samples_batch(sk.handle, _ptr(X), C.c_int64(B), C.byref(pc), _ptr(indices),
                                                   _ptr(out.counts), _ptr(out.support), _ptr(out.values),
                                                   _ptr(out.candidates), _ptr(out.mu), C.c_void_p(stream)))
    return out


def transform(sk: Sketch, x, p: StreamParams) -> TransformResult:
    """stream.hpp:272-275 for one vector (seed = p.seed)."""
    x = np.asarray(x)
    if x.ndim != 1:
        raise ValueError("transform: x must be a vector")
    r = transform_batch(sk, x.reshape(1, -1), p, candidates=True, mu=True)
    return r.result(0, p.J * p.K)


def transform_with_samples(sk: Sketch, x, p: StreamParams, indices) -> TransformResult:
    """stream.hpp:197-268 for one vector with pre-drawn indices."""
    x = np.asarray(x)
    r = transform_with_samples_batch(sk, x.reshape(1, -1), p, np.asarray(indices, dtype=np.int64).reshape(1, -1),
                                     candidates=True, mu=True)
    return r.result(0, p.J * p.K)


# -------------------------------------------------------- public helpers ----
def inner_product_with_design(x, k: int, ell: int, device: int = 0) -> float:
    """stream.hpp:109-121 on the GPU: s_ell^T x (Kerdock: the reference's Gray-code walk, bit-exact)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = C.c_double()
    _check(lib().fstg_inner_product_with_design(C.c_int(k), _ptr(x), C.c_int64(x.size), C.c_int64(ell),
                                                C.byref(out), C.c_int(device)))
    return out.value


def median_of_means(samples, J: int, K: int, device: int = 0) -> np.ndarray:
    """stream.hpp:147-155 on the GPU: samples (m, J*K), batch b = columns [b*J, (b+1)*J)."""
    samples = np.asarray(samples, dtype=np.float64)
    if samples.ndim != 2 or J < 1 or K < 1 or samples.shape[1] != J * K:
        raise ValueError("median_of_means: samples must have J*K columns")
    m = samples.shape[0]
    cols = np.ascontiguousarray(samples.T)          # row j = column j of the reference's m x N matrix
    out = np.zeros(m)
    _check(lib().fstg_median_of_means(_ptr(cols), C.c_int64(m), C.c_int64(J), C.c_int64(K), _ptr(out),
                                      C.c_int(device)))
    return out


def hard_threshold(v, eps: float, device: int = 0) -> np.ndarray:
    """stream.hpp:158-162 on the GPU (|t| = eps kept)."""
    v = np.ascontiguousarray(v, dtype=np.float64)
    out = np.zeros_like(v)
    _check(lib().fstg_hard_threshold(_ptr(v), C.c_int64(v.size), C.c_double(eps), _ptr(out), C.c_int(device)))
    return out


def projected_design_column(k: int, n: int, ell: int, device: int = 0) -> np.ndarray:
    """kerdock.hpp:156-167 on the GPU: s_ell (n entries)."""
    out = np.zeros(n)
    _check(lib().fstg_projected_design_column(C.c_int(k), C.c_int64(n), C.c_int64(ell), _ptr(out), C.c_int(device)))
    return out


# ------------------------------------------------------- design verifiers ----
VERIFY_REFERENCE = 0   # the reference's policy: exhaustive for k <= 6, sampled above (same seeds)
VERIFY_EXHAUSTIVE = 1  # every basis pair / every column pair, any k <= cap


class _MubReport(C.Structure):
    _fields_ = [("max_within_gram_dev", C.c_double), ("min_cross_sq", C.c_double), ("max_cross_sq", C.c_double),
                ("max_cross_dev", C.c_double), ("exhaustive", C.c_int32), ("reserved", C.c_int32),
                ("basis_pairs", C.c_int64)]


class _MomentReport(C.Structure):
    _fields_ = [("m1", C.c_double), ("m2", C.c_double), ("exact", C.c_int32), ("reserved", C.c_int32),
                ("pairs", C.c_int64)]


@dataclass
class MubReport:
    """kerdock.hpp:199-208"""
    max_within_gram_dev: float
    min_cross_sq: float
    max_cross_sq: float
    max_cross_dev: float
    exhaustive: bool
    basis_pairs: int

    def passed(self, tol: float) -> bool:
        return self.max_within_gram_dev <= tol and self.max_cross_dev <= tol


@dataclass
class MomentReport:
    """kerdock.hpp:261-266"""
    m1: float
    m2: float
    exact: bool
    pairs: int


def verify_mub(k: int, cap: int = 8, policy: int = VERIFY_REFERENCE, device: int = 0) -> MubReport:
    """kerdock.hpp:213-256 on the GPU (k > cap raises ValueError like the reference's invalid_argument)."""
    r = _MubReport()
    _check(lib().fstg_verify_mub(C.c_int(k), C.c_int(cap), C.c_int(policy), C.c_int(device), C.byref(r)))
    return MubReport(r.max_within_gram_dev, r.min_cross_sq, r.max_cross_sq, r.max_cross_dev, bool(r.exhaustive),
                     int(r.basis_pairs))


def verify_design_moments(k: int, cap: int = 8, policy: int = VERIFY_REFERENCE, device: int = 0) -> MomentReport:
    """kerdock.hpp:301-315 on the GPU."""
    r = _MomentReport()
    _check(lib().fstg_verify_design_moments(C.c_int(k), C.c_int(cap), C.c_int(policy), C.c_int(device),
                                            C.byref(r)))
    return MomentReport(r.m1, r.m2, bool(r.exact), int(r.pairs))


def design_moment_target(d: int, k: int) -> float:
    """kerdock.hpp:267-276: c_{d,k} = 1*3*...*(2k-1) / (d (d+2) ... (d+2(k-1)))."""
    return float(lib().fstg_design_moment_target(C.c_int64(d), C.c_int(k)))


def verify_kerdock_set(k: int, device: int = 0):
    """cli.hpp:45-60: (all matrices symmetric with zero diagonal, rank-deficient pair-sum count)."""
    skew, bad = C.c_int(), C.c_int64()
    _check(lib().fstg_verify_kerdock_set(C.c_int(k), C.c_int(device), C.byref(skew), C.byref(bad)))
    return bool(skew.value), int(bad.value)


# -------------------------------------------------------------- profiling ----
def profile_enable(on: bool = True) -> None:
    _check(lib().fstg_profile_enable(C.c_int(1 if on else 0)))


def profile_reset() -> None:
    _check(lib().fstg_profile_reset())


def profile_read(name: str):
    ms, n = C.c_double(), C.c_int64()
    _check(lib().fstg_profile_read(name.encode(), C.byref(ms), C.byref(n)))
    return ms.value, n.value


def set_pool_retain(retain: bool) -> None:
    """Keep the library pool's large transient buffers cached across calls (see fstg_set_pool_retain)."""
    _check(lib().fstg_set_pool_retain(C.c_int(1 if retain else 0)))


def launch_count() -> int:
    n = C.c_int64()
    _check(lib().fstg_launch_count(C.byref(n)))
    return n.value
