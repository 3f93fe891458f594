"""The oracle restatement pinned against the REFERENCE ITSELF.

oracle/_ref/libfst_ref.so is the reference's own sketch.hpp / stream.hpp / kerdock.hpp
code, compiled unmodified from /root/reference against the Eigen-API shim
(oracle/eigen_shim, oracle/ref_capi.cpp; `make -C oracle ref`). These CPU tests run
it beside the oracle (oracle/fst_oracle.cpp) on the same inputs:
  - preprocess (sketch.hpp:149-211): every sketch column bit-identical;
  - draw_samples (stream.hpp:173-182): identical indices;
  - transform (stream.hpp:197-275): identical mu (bit for bit), candidate set and support,
    and refined values (the shim's sequential dot: bit-identical here, 1e-12 allowed by
    north_star for fp64);
  - the draw_and_gather form on a sketch without materialised columns (the form bench.py
    times at n = 4096) equals the full-sketch transform;
  - choose_params (stream.hpp:58-69).
Edge cases follow the reference's tests (proj/tests/test_stream.cpp, test_sketch.cpp):
non-square A with padding (n < d), identity-block draws, widen*s >= m, even K (median of
an even count), J = 1, K = 1.
"""
import numpy as np
import pytest

from oracle import oracle as orc
from oracle import refimpl as ref

pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref/libfst_ref.so not built "
                                                            "(make -C oracle ref needs /root/reference)")


def _rect(m, n, seed):
    g = orc.rng_gaussian(seed, m * n).reshape(m, n)
    return g / np.sqrt(n)


@pytest.mark.parametrize("m,n", [(16, 16), (64, 64), (256, 256), (100, 50), (40, 200), (1, 4)])
def test_preprocess_columns_bit_identical(m, n):
    a = _rect(m, n, 1000 + m + n)
    r = ref.preprocess(a, threads=4)
    o = orc.preprocess(a)
    assert (r.m, r.n, r.L) == (m, n, o.columns().shape[0])
    assert r.columns().tobytes() == o.columns().tobytes()
    assert r.row_norm_max == pytest.approx(float(np.max(np.linalg.norm(a, axis=1))), rel=1e-14)


CASES = [
    # (m, n, s, eps, J, K, widen)
    (256, 256, 8, 0.1, 375, 2, 10),      # config-1 shape at the bench's J, K
    (64, 64, 4, 0.1, 60, 3, 10),
    (64, 64, 4, 0.1, 17, 4, 10),         # even K: median = mean of the middle pair
    (64, 64, 4, 0.05, 1, 1, 10),         # J = K = 1
    (100, 50, 5, 0.05, 40, 3, 10),       # non-square, padded n < d
    (40, 200, 3, 0.1, 25, 5, 2),
    (32, 32, 8, 0.1, 20, 3, 10),         # widen*s >= m: every row is a candidate
]


@pytest.mark.parametrize("m,n,s,eps,J,K,widen", CASES)
def test_transform_matches_reference(m, n, s, eps, J, K, widen):
    a = orc.gen_orthogonal(n, 900 + n)[:m] if m <= n else _rect(m, n, 77)
    rs = ref.preprocess(a, threads=2)
    os_ = orc.preprocess(a)
    cols = os_.columns()
    bare = ref.sketch_without_columns(a)
    for v in range(4):
        x = orc.rng_gaussian(orc.gen_seed(v) ^ 0x55, n)
        x /= np.linalg.norm(x)
        p = orc.StreamParams(epsilon=eps, s=s, J=J, K=K, widen=widen, seed=orc.stream_seed(v))
        idx = ref.draw_samples(rs, p)
        assert np.array_equal(idx, orc.draw_samples(rs.L, p))
        r = ref.transform(rs, x, p)
        o = orc.transform(os_, x, p)
        assert r.mu.tobytes() == o.mu.tobytes()
        assert r.candidate_set.tolist() == o.candidate_set.tolist()
        assert r.support.tolist() == o.support.tolist()
        np.testing.assert_allclose(r.values, o.values, rtol=1e-12, atol=1e-15)
        g = ref.transform(bare, x, p, gathered=cols[idx])
        assert g.mu.tobytes() == r.mu.tobytes()
        assert g.support.tolist() == r.support.tolist()


def test_identity_block_draws_covered():
    """k = 4: L = 16 * 9 = 144, identity block = the last 16 columns; 300 draws hit it."""
    a = orc.gen_orthogonal(16, 3)
    rs, os_ = ref.preprocess(a), orc.preprocess(a)
    x = a.T @ np.eye(16)[2]
    p = orc.StreamParams(epsilon=0.1, s=1, J=100, K=3, seed=11)
    idx = ref.draw_samples(rs, p)
    assert np.any(idx >= 144 - 16)
    r, o = ref.transform(rs, x, p), orc.transform(os_, x, p)
    assert r.mu.tobytes() == o.mu.tobytes() and r.support.tolist() == o.support.tolist() == [2]


@pytest.mark.parametrize("rn,gamma,eta,m", [(1.0, 0.05, 0.1, 256), (1.7, 0.01, 0.5, 4096), (0.3, 1.0, 1.0, 1)])
def test_choose_params_matches_reference(rn, gamma, eta, m):
    assert ref.choose_params(rn, gamma, eta, m) == orc.choose_params(rn, gamma, eta, m)


def test_reference_errors_map_to_exceptions():
    a = orc.gen_orthogonal(16, 3)
    rs = ref.preprocess(a)
    with pytest.raises(ValueError):
        ref.transform(rs, np.zeros(15), orc.StreamParams(epsilon=0.1, s=1, J=4, K=1, seed=1))
    with pytest.raises(ValueError):
        ref.transform(rs, np.zeros(16), orc.StreamParams(epsilon=0.1, s=1, J=0, K=1, seed=1))


def test_bench_gathered_counts_match_oracle():
    """The timed loop bench.py runs as the reference arm: same support counts as the oracle's."""
    n = 64
    a = orc.gen_orthogonal(n, 5)
    os_ = orc.preprocess(a)
    cols = os_.columns()
    P = 6
    X = np.stack([orc.gen_exact_sparse(a, 4, orc.gen_seed(v))[0] for v in range(P)])
    seeds = np.array([orc.stream_seed(v) for v in range(P)], dtype=np.uint64)
    p = orc.StreamParams(epsilon=0.1, s=4, J=60, K=3)
    gathered = np.stack([cols[orc.draw_samples(cols.shape[0], orc.StreamParams(epsilon=0.1, s=4, J=60, K=3,
                                                                                 seed=int(sd)))] for sd in seeds])
    counts, secs = ref.bench_gathered(a, X, p, seeds, gathered, threads=2, total=3 * P)
    counts_o, _ = orc.bench_gathered(a, X, p, seeds, gathered, cols.shape[0], 2, P)
    assert counts.tolist() == counts_o.tolist() and secs > 0
