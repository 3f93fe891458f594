"""FSTK persistence (sketch.hpp:213-302): the oracle restatement against the
reference's own save/load tests (test_sketch.cpp:146-202) on CPU, and the GPU
library's save/load against the oracle (byte-compatible files, the same four
error classes) on a B200."""
import os

import numpy as np
import pytest


def _rand(m, n, seed):
    return np.random.default_rng(seed).standard_normal((m, n))


def _corrupt(path, offset, data):
    with open(path, "r+b") as f:
        f.seek(offset)
        f.write(data)


# --------------------------------------------------------------- oracle ----
def test_oracle_roundtrip_bit_exact(orc, tmp_path):  # test_sketch.cpp:146-164
    sk = orc.preprocess(_rand(8, 16, 9))
    path = str(tmp_path / "rt.fstk")
    orc.save(sk, path)
    back = orc.load(path)
    assert (back.m, back.n, back.k, back.L) == (sk.m, sk.n, sk.k, sk.L)
    assert back.row_norm_max == sk.row_norm_max
    assert back.columns().tobytes() == sk.columns().tobytes()
    assert os.path.getsize(path) == 49 + 8 * sk.m * sk.L + 8 * sk.m * sk.n


def _error_cases(load, save_fn, tmp_path, errors):
    path = str(tmp_path / "err.fstk")
    save_fn(path)
    size = os.path.getsize(path)
    _corrupt(path, 0, b"NOPE")
    with pytest.raises(errors.MagicMismatchError):
        load(path)
    save_fn(path)
    _corrupt(path, 4, bytes([3, 0, 0, 0]))
    with pytest.raises(errors.VersionUnsupportedError):
        load(path)
    save_fn(path)
    os.truncate(path, size - 17)
    with pytest.raises(errors.TruncatedPayloadError):
        load(path)
    os.truncate(path, 10)
    with pytest.raises(errors.TruncatedPayloadError):
        load(path)
    save_fn(path)
    _corrupt(path, 8 + 2 * 8, bytes([3, 0, 0, 0, 0, 0, 0, 0]))  # k = 3
    with pytest.raises(errors.MalformedHeaderError):
        load(path)
    save_fn(path)
    with open(path, "ab") as f:
        f.write(b"\0" * 8)
    with pytest.raises(errors.MalformedHeaderError):
        load(path)
    with pytest.raises(errors.IoError):
        load(str(tmp_path / "missing.fstk"))


def test_oracle_load_errors(orc, tmp_path):  # test_sketch.cpp:166-202
    sk = orc.preprocess(_rand(3, 4, 10))
    _error_cases(orc.load, lambda p: orc.save(sk, p), tmp_path, orc)


# ------------------------------------------------------------------ GPU ----
@pytest.fixture(scope="module")
def fst():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2105_05879_b200 import fst
    return fst


@pytest.mark.gpu
def test_gpu_save_loads_in_oracle(fst, orc, tmp_path):
    a = _rand(40, 50, 3)
    path = str(tmp_path / "gpu.fstk")
    fst.save(fst.preprocess(a), path, version=1)
    back = orc.load(path)
    ref = orc.preprocess(a)
    assert back.columns().tobytes() == ref.columns().tobytes()
    assert back.row_norm_max == pytest.approx(ref.row_norm_max, rel=1e-14)
    with open(path, "rb") as f:
        assert f.read(4) == b"FSTK"


@pytest.mark.gpu
def test_oracle_save_loads_on_gpu(fst, orc, tmp_path):
    a = _rand(33, 64, 4)
    ref = orc.preprocess(a)
    path = str(tmp_path / "orc.fstk")
    orc.save(ref, path)
    sk = fst.load(path)  # fp64 kept
    cols = ref.columns()
    for ell in range(0, sk.L, 7):
        assert sk.column(ell).tobytes() == cols[ell].tobytes()
    x = np.random.default_rng(1).standard_normal(64)
    p = fst.StreamParams(epsilon=0.05, s=3, J=40, K=3, seed=5)
    g = fst.transform(sk, x, p)
    r = orc.transform(ref, x, orc.StreamParams(epsilon=0.05, s=3, J=40, K=3, seed=5))
    assert np.array_equal(g.mu, r.mu) and g.support.tolist() == r.support.tolist()
    sk32 = fst.load(path, dtype=np.float32)  # rounded on the GPU
    for ell in range(0, sk32.L, 11):
        assert np.array_equal(sk32.column(ell), cols[ell].astype(np.float32))


@pytest.mark.gpu
def test_gpu_v2_float32_roundtrip(fst, orc, tmp_path):
    a = _rand(17, 200, 5).astype(np.float32)
    sk = fst.preprocess(a)
    path = str(tmp_path / "v2.fstk")
    fst.save(sk, path, version=2)
    assert os.path.getsize(path) == 49 + 4 * sk.m * sk.L + 4 * sk.m * sk.n
    back = fst.load(path)
    assert back.dtype == np.float32 and back.row_norm_max() == sk.row_norm_max()
    for ell in range(0, sk.L, 13):
        assert back.column(ell).tobytes() == sk.column(ell).tobytes()
    with pytest.raises(orc.VersionUnsupportedError):
        orc.load(path)  # the reference format is float64-only
    with pytest.raises(ValueError):
        fst.save(fst.preprocess(a.astype(np.float64)), path, version=2)


@pytest.mark.gpu
def test_gpu_load_errors_and_no_matrix(fst, orc, tmp_path):
    sk = orc.preprocess(_rand(3, 4, 10))
    _error_cases(fst.load, lambda p: orc.save(sk, p), tmp_path, fst)
    path = str(tmp_path / "noa.fstk")
    orc.save(sk, path, with_a=False)
    g = fst.load(path)
    assert g.row_norm_max() == 0.0
    with pytest.raises(fst.NoMatrixError):
        fst.transform(g, np.ones(4), fst.StreamParams(epsilon=0.1, s=1, J=2, K=2))
    with pytest.raises(fst.NoMatrixError):
        g.embedded_matrix()


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_gpu_load_rows_longer_than_staging_chunk(tmp_path, dtype):
    """A reference FSTK v1 file whose m (8,388,613) makes one column longer than the 64 MiB
    pinned / staging chunk: the load reads element pieces, never past either
    buffer, and save writes the same bytes back. Sparse file: zeros except a few marked values
    at the piece boundaries."""
    import struct
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2105_05879_b200 import fst
    m, n, k = 8388613, 3, 2
    d, L = 4, 12
    path = str(tmp_path / "tall.fstk")
    header = b"FSTK" + struct.pack("<IQQQQQB", 1, m, n, k, d, L, 1)
    payload = 8 * m * L + 8 * m * n
    with open(path, "wb") as f:
        f.write(header)
        f.truncate(49 + payload)
    marks = {(0, 0): 1.5, (0, 8388607): -2.25, (0, 8388608): 3.0, (0, m - 1): 4.5, (1, 0): -6.0, (11, m - 1): 7.0}
    for (col, row), val in marks.items():
        _corrupt(path, 49 + 8 * (col * m + row), struct.pack("<d", val))
    _corrupt(path, 49 + 8 * m * L + 8 * (m * n - 1), struct.pack("<d", 9.0))   # last entry of A
    sk = fst.load(path, dtype=dtype)
    assert (sk.m, sk.n, sk.L) == (m, n, L)
    for (col, row), val in marks.items():
        c = sk.column(col)
        assert c[row] == val, (col, row)
    assert np.count_nonzero(sk.column(0)) == 4
    assert sk.embedded_matrix()[-1, -1] == 9.0
    if dtype == np.float64:
        out = str(tmp_path / "tall2.fstk")
        fst.save(sk, out, version=1)
        with open(path, "rb") as a, open(out, "rb") as b:
            while True:
                x, y = a.read(1 << 24), b.read(1 << 24)
                assert x == y
                if not x:
                    break
    sk.close()
