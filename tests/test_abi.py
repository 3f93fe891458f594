"""CPU tests of the C-ABI library: it loads, exports every symbol include/fst_b200.h
declares, its host-side design logic matches the oracle bit-exactly, and the
compute entry points fail loudly (no CPU fallback) when no B200 is present."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fst_b200.h")


@pytest.fixture(scope="module")
def fst():
    from paper_2105_05879_b200 import fst
    if not os.path.exists(fst.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    return fst


def _declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(fstg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(fst):
    lib = C.CDLL(fst.LIB_PATH)
    declared = _declared_functions()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(fst.EXPORTED) == declared


def test_sm100a_cubin_only(fst):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", fst.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", ""))


def test_design_params_and_log2(fst, orc):
    for n in [1, 3, 4, 5, 16, 17, 64, 65, 256, 1024, 4096, 16384]:
        assert fst.even_log2_ceil(n) == orc.even_log2_ceil(n)
    for k in (2, 4, 6, 8, 10, 12, 14, 16):
        assert fst.design_params(k) == orc.design_params(k)
    for bad in (0, 3, 18):
        with pytest.raises(ValueError):
            fst.design_params(bad)
    with pytest.raises(ValueError):
        fst.even_log2_ceil(0)


@pytest.mark.parametrize("k", [2, 4, 6, 8, 10, 12])
def test_kerdock_matrices_match_oracle(fst, orc, k):
    d, _ = orc.design_params(k)
    for s in range(d // 2):                      # every basis (k = 12: 2048)
        assert fst.kerdock_matrix(k, s).tolist() == orc.kerdock_matrix(k, s).tolist(), (k, s)


def test_kerdock_k14_all_bases(fst, orc):
    for s in range(8192):                        # the config-4 design: every basis
        assert fst.kerdock_matrix(14, s).tolist() == orc.kerdock_matrix(14, s).tolist(), s
    with pytest.raises(ValueError):
        fst.kerdock_matrix(4, 8)


def test_choose_params_matches_reference(fst, orc):
    assert fst.choose_params(1.0, 1.0, 1.0, 1) == (30, 1)
    assert fst.choose_params(1.0, 0.5, 0.01, 4096) == (119, 26)
    rng = np.random.default_rng(5)
    for _ in range(200):
        r, g, eta, m = rng.uniform(0.1, 3), rng.uniform(0.01, 2), rng.uniform(0.01, 1), int(rng.integers(1, 10**5))
        assert fst.choose_params(r, g, eta, m) == orc.choose_params(r, g, eta, m)
    for bad in [(1.0, 0.0, 0.5, 16), (1.0, 0.5, 0.0, 16), (1.0, 0.5, 1.5, 16), (1.0, 0.5, 0.5, 0)]:
        with pytest.raises(ValueError):
            fst.choose_params(*bad)


def test_candidate_count(fst, orc):
    for s, w, m in [(32, 10, 4096), (8, 10, 256), (2, 8, 16), (4, 10, 32), (10**15, 10, 64), (3, 1, 5)]:
        assert fst.candidate_count(s, w, m) == orc.candidate_count(s, w, m)


def test_param_validation(fst):
    P = fst.StreamParams
    P(epsilon=0.1, s=1, J=2, K=2).validate()
    for kw in [dict(epsilon=0.0), dict(epsilon=0.1, delta=0.2), dict(epsilon=0.1, s=0), dict(epsilon=0.1, J=0),
               dict(epsilon=0.1, K=0), dict(epsilon=0.1, widen=0), dict(epsilon=0.1, delta=-1.0)]:
        with pytest.raises(ValueError):
            P(**{**dict(s=1, J=2, K=2), **kw}).validate()
    with pytest.raises(OverflowError):
        P(epsilon=0.1, s=1, J=(2**63 - 1) // 2, K=3).validate()


def test_no_cpu_fallback_without_gpu(fst):
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    assert fst.device_count() == 0
    with pytest.raises(fst.CudaError):
        fst.preprocess(np.eye(4))


def test_python_buffer_validation():
    """The Python mirror rejects buffers the C-ABI would read or write past:
    short or mistyped seeds, mis-shaped outputs, outputs on the wrong side."""
    from paper_2105_05879_b200 import fst
    B, want, m = 4, 10, 32
    fst._check_seeds(np.zeros(B, dtype=np.uint64), B)
    fst._check_seeds(np.zeros(B, dtype=np.int64), B)
    for bad in (np.zeros(B - 1, dtype=np.uint64), np.zeros(B, dtype=np.int32), np.zeros((B, 1), dtype=np.int64)):
        with pytest.raises(ValueError):
            fst._check_seeds(bad, B)
    ok = fst.BatchResult(np.zeros(B, np.int32), np.zeros((B, want), np.int32), np.zeros((B, want), np.float32),
                         np.zeros((B, want), np.int32), np.zeros((B, m), np.float32))
    fst._check_outputs(ok, B, want, m, np.float32, None)
    bad_cases = [
        fst.BatchResult(np.zeros(B - 1, np.int32), ok.support, ok.values),
        fst.BatchResult(ok.counts, np.zeros((B, want - 1), np.int32), ok.values),
        fst.BatchResult(ok.counts, ok.support, np.zeros((B, want), np.float64)),
        fst.BatchResult(ok.counts, ok.support, ok.values, np.zeros((B, want), np.int64)),
        fst.BatchResult(ok.counts, ok.support, ok.values, None, np.zeros((B, m + 1), np.float32)),
    ]
    for out in bad_cases:
        with pytest.raises(ValueError):
            fst._check_outputs(out, B, want, m, np.float32, None)
    with pytest.raises(ValueError):  # host outputs for device inputs
        fst._check_outputs(ok, B, want, m, np.float32, "cuda:0")
