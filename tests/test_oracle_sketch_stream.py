"""Pins the oracle's preprocess / transform against proj/tests/test_sketch.cpp,
test_stream.cpp and acceptance.cpp (known answers and properties). CPU only."""
import numpy as np
import pytest


def _rand(m, n, seed):
    return np.random.default_rng(seed).standard_normal((m, n))


def _orthogonal(n, seed):
    q, r = np.linalg.qr(np.random.default_rng(seed).standard_normal((n, n)))
    return q * np.sign(np.diag(r))


def _unit(n, seed):
    x = np.random.default_rng(seed).standard_normal(n)
    return x / np.linalg.norm(x)


def _naive_column(orc, a, k, ell):  # test_sketch.cpp:24-27
    return a @ orc.projected_design_column(k, a.shape[1], ell)


# ----------------------------------------------------------- test_sketch.cpp --
def test_even_log2_ceil(orc):  # test_sketch.cpp:35-45
    for n, k in [(1, 2), (3, 2), (4, 2), (5, 4), (16, 4), (17, 6), (64, 6), (65, 8)]:
        assert orc.even_log2_ceil(n) == k
    with pytest.raises(ValueError):
        orc.even_log2_ceil(0)


def test_identity_reproduces_design(orc):  # test_sketch.cpp:47-60
    sk = orc.preprocess(np.eye(16))
    assert (sk.k, sk.L) == (4, 144)
    assert sk.row_norm_max == pytest.approx(1.0)
    cols = sk.columns()
    for ell in range(sk.L):
        assert np.max(np.abs(cols[ell] - orc.projected_design_column(4, 16, ell))) <= 1e-12
        if ell < 8 * 16:
            assert np.all(np.abs(cols[ell]) == 1.0)


def test_k4_columns_vs_naive(orc):  # test_sketch.cpp:62-68
    a = _rand(8, 16, 99)
    sk = orc.preprocess(a)
    cols = sk.columns()
    for ell in range(sk.L):
        assert np.max(np.abs(cols[ell] - _naive_column(orc, a, 4, ell))) <= 1e-9


@pytest.mark.parametrize("m,n,seed", [(5, 13, 1), (3, 50, 2), (7, 4, 3)])
def test_padding_vs_naive(orc, m, n, seed):  # test_sketch.cpp:70-82
    a = _rand(m, n, seed)
    sk = orc.preprocess(a)
    rng = np.random.default_rng(seed * 31)
    cols = sk.columns()
    for ell in rng.integers(0, sk.L, size=200):
        assert np.max(np.abs(cols[ell] - _naive_column(orc, a, sk.k, int(ell)))) <= 1e-9


def test_ones_row(orc):  # test_sketch.cpp:84-88
    assert orc.preprocess(np.ones((1, 4))).column(0)[0] == pytest.approx(4.0)


def test_mean_identity_and_linearity(orc):  # test_sketch.cpp:90-115
    a = _rand(6, 13, 4)
    sk = orc.preprocess(a)
    x = _unit(13, 5)
    cols = sk.columns()
    mean = sum(cols[ell] * (orc.projected_design_column(sk.k, 13, ell) @ x) for ell in range(sk.L)) / sk.L
    assert np.max(np.abs(mean - a @ x)) <= 1e-9
    a2 = _rand(4, 7, 6)
    c1, c2 = orc.preprocess(a2).columns(), orc.preprocess(3.5 * a2).columns()
    assert np.max(np.abs(3.5 * c1 - c2)) <= 1e-9


def test_bounds_and_zero_identity(orc):  # test_sketch.cpp:117-126
    a = _rand(5, 13, 7)
    sk = orc.preprocess(a)
    with pytest.raises(IndexError):
        sk.column(sk.L)
    with pytest.raises(IndexError):
        sk.column(-1)
    assert not sk.column(sk.L - 1).any()
    assert np.max(np.abs(sk.column(0) - a @ np.ones(13))) <= 1e-9


def test_rejects_empty_and_nonfinite(orc):  # test_sketch.cpp:128-133
    with pytest.raises(ValueError):
        orc.preprocess(np.zeros((0, 0)))
    bad = np.ones((2, 2))
    bad[0, 1] = np.nan
    with pytest.raises(ValueError):
        orc.preprocess(bad)


def test_thread_count_bit_identity(orc):  # test_sketch.cpp:135-144
    a = _rand(9, 16, 8)
    c1 = orc.preprocess(a, threads=1).columns().copy()
    c4 = orc.preprocess(a, threads=4).columns().copy()
    assert c1.tobytes() == c4.tobytes()


def test_acceptance_sketch_oracle(orc):  # acceptance.cpp:101-116
    g = orc.rng_gaussian(20240817, 8 * 16).reshape(8, 16)
    sk = orc.preprocess(g)
    cols = sk.columns()
    worst = max(np.max(np.abs(cols[ell] - _naive_column(orc, g, 4, ell))) for ell in range(sk.L))
    assert worst <= 1e-9


# ----------------------------------------------------------- test_stream.cpp --
def test_choose_params_fixed(orc):  # test_stream.cpp:40-64
    assert orc.choose_params(1.0, 1.0, 1.0, 1) == (30, 1)
    assert orc.choose_params(1.0, 0.5, 0.01, 4096) == (119, 26)
    for bad in (0.0, -1.0):
        with pytest.raises(ValueError):
            orc.choose_params(1.0, bad, 0.5, 16)
    for g in (0.1, 0.25, 0.7, 1.3):
        j1, k1 = orc.choose_params(1.0, g, 0.5, 64)
        j2, k2 = orc.choose_params(1.0, 2 * g, 0.5, 64)
        assert k1 == k2 and j1 // 4 <= j2 <= j1 // 4 + 1
    for eta in (0.0, 1.5):
        with pytest.raises(ValueError):
            orc.choose_params(1.0, 0.5, eta, 16)
    orc.choose_params(1.0, 0.5, 1.0, 16)
    with pytest.raises(ValueError):
        orc.choose_params(1.0, 0.5, 0.5, 0)


def test_inner_product_fixed(orc):  # test_stream.cpp:66-84
    x = np.array([1.0, 2, 3, 4])
    assert orc.inner_product_with_design(x, 2, 0) == pytest.approx(10.0)
    assert orc.inner_product_with_design(x, 2, 4) == pytest.approx(2.0)
    short = np.array([1.0, 2, 3])
    assert orc.inner_product_with_design(short, 2, 8 + 3) == 0.0
    assert orc.inner_product_with_design(short, 2, 8 + 1) == pytest.approx(4.0)


def test_inner_product_vs_materialized(orc):  # test_stream.cpp:86-102
    rng = np.random.default_rng(100)
    for k in (2, 4, 6):
        d, L = orc.design_params(k)
        for n in (d, d - 3, 1 + d // 3):
            x = rng.standard_normal(n)
            for ell in rng.integers(0, L, size=100):
                expect = orc.projected_design_column(k, n, int(ell)) @ x
                assert orc.inner_product_with_design(x, k, int(ell)) == pytest.approx(expect, rel=1e-12, abs=1e-12)


def test_median_of_means_fixed(orc):  # test_stream.cpp:104-137
    assert orc.median_of_means(np.array([[1.0, 2, 3, 6]]), 4, 1)[0] == pytest.approx(3.0)
    assert orc.median_of_means(np.array([[1.0, 3, 2, 4, 100, -100]]), 2, 3)[0] == pytest.approx(2.0)
    with pytest.raises(ValueError):
        orc.median_of_means(np.array([[1.0, 3, 2, 4, 100, -100]]), 2, 2)
    samples = np.random.default_rng(33).standard_normal((5, 12))
    assert np.max(np.abs(orc.median_of_means(samples, 6, 2) - samples.mean(axis=1))) <= 1e-14
    assert orc.median_of_batch_means(np.array([[7.0, 1, 3, 100]]))[0] == pytest.approx(5.0)
    assert orc.median_of_batch_means(np.array([[9.0, 1, 3, 100, -4]]))[0] == pytest.approx(3.0)


def test_hard_threshold(orc):  # test_stream.cpp:139-160
    h = orc.hard_threshold(np.array([0.6, -0.3, 0.5]), 0.5)
    assert h.tolist() == [0.6, 0.0, 0.5]


def _params(orc, **kw):
    p = orc.StreamParams()
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def test_widen_covers_all_rows_is_exact(orc):  # test_stream.cpp:162-189
    a = _orthogonal(16, 1)
    sk = orc.preprocess(a)
    x = _unit(16, 2)
    res = orc.transform(sk, x, _params(orc, epsilon=0.2, s=2, widen=8, J=3, K=2, seed=42))
    ax = a @ x
    expect = np.nonzero(np.abs(ax) >= 0.2)[0]
    assert len(res.candidate_set) == 16
    assert res.support.tolist() == expect.tolist()
    np.testing.assert_allclose(res.values, ax[expect], rtol=1e-12)


def test_zero_vector(orc):  # test_stream.cpp:191-202
    sk = orc.preprocess(_orthogonal(16, 3))
    res = orc.transform(sk, np.zeros(16), _params(orc, epsilon=0.1, s=2, J=5, K=2))
    assert len(res.support) == 0 and len(res.values) == 0
    assert not res.mu.any()


def test_one_spike_recovery(orc):  # test_stream.cpp:204-225
    a = _orthogonal(16, 4)
    sk = orc.preprocess(a)
    x = a[0].copy()
    ok = 0
    for seed in range(100):
        r = orc.transform(sk, x, _params(orc, epsilon=0.5, s=1, widen=10, J=500, K=3, seed=seed))
        ok += int(r.support.tolist() == [0] and abs(r.values[0] - 1.0) <= 1e-10)
    assert ok == 100


def test_soundness(orc):  # test_stream.cpp:227-249
    a = _orthogonal(32, 5)
    sk = orc.preprocess(a)
    x = _unit(32, 6)
    ax = a @ x
    r = orc.transform(sk, x, _params(orc, epsilon=0.05, s=4, J=40, K=3, seed=7))
    assert len(r.candidate_set) == 32
    assert np.all(np.abs(r.values - ax[r.support]) <= 1e-12)
    assert np.all(np.abs(r.values) >= 0.05)
    assert set(r.support.tolist()) <= set(r.candidate_set.tolist())


def test_unbiased_sweep(orc):  # test_stream.cpp:251-263
    a = _orthogonal(16, 8)
    sk = orc.preprocess(a)
    x = _unit(16, 9)
    cols = sk.columns()
    mean = sum(cols[ell] * orc.inner_product_with_design(x, sk.k, ell) for ell in range(sk.L)) / sk.L
    assert np.max(np.abs(mean - a @ x)) <= 1e-9


def test_determinism_and_fused_vs_materialized(orc):  # test_stream.cpp:290-340
    a = _orthogonal(32, 10)
    sk = orc.preprocess(a)
    x = _unit(32, 11)
    p = _params(orc, epsilon=0.05, s=3, J=25, K=4, seed=1234)
    r1, r2 = orc.transform(sk, x, p), orc.transform(sk, x, p)
    r3 = orc.transform_with_samples(sk, x, p, orc.draw_samples(sk.L, p))
    for r in (r2, r3):
        assert r.support.tolist() == r1.support.tolist()
        assert r.values.tobytes() == r1.values.tobytes()
        assert r.candidate_set.tolist() == r1.candidate_set.tolist()
        assert r.mu.tobytes() == r1.mu.tobytes()
    a = _orthogonal(16, 12)
    sk = orc.preprocess(a)
    x = _unit(16, 13)
    p = _params(orc, epsilon=0.1, s=2, J=11, K=3, seed=99)
    idx = orc.draw_samples(sk.L, p)
    cols = sk.columns()
    samples = np.stack([cols[ell] * orc.inner_product_with_design(x, sk.k, int(ell)) for ell in idx], axis=1)
    direct = orc.median_of_means(samples, p.J, p.K)
    r = orc.transform_with_samples(sk, x, p, idx)
    assert np.max(np.abs(r.mu - direct)) <= 1e-12


def test_validation_errors(orc):  # test_stream.cpp:382-401
    sk = orc.preprocess(_orthogonal(16, 14))
    with pytest.raises(ValueError):
        orc.transform(sk, np.zeros(15), _params(orc, epsilon=0.1, s=1, J=2, K=2))
    with pytest.raises(ValueError):
        orc.transform(sk, np.zeros(16), _params(orc, epsilon=0.0, s=1, J=2, K=2))
    with pytest.raises(ValueError):
        orc.transform(sk, np.zeros(16), _params(orc, epsilon=0.1, delta=0.2, s=1, J=2, K=2))
    with pytest.raises(OverflowError):
        _params(orc, epsilon=0.1, s=1, J=(2**63 - 1) // 2, K=3).validate()


def test_gen_orthogonal_and_exact_sparse(orc):  # generators.hpp:20-55
    a = orc.gen_orthogonal(64, 777)
    assert np.max(np.abs(a @ a.T - np.eye(64))) <= 1e-12
    x, truth = orc.gen_exact_sparse(a, 8, 5000)
    assert np.count_nonzero(truth) == 8
    assert np.allclose(np.abs(truth[truth != 0]), 1 / np.sqrt(8))
    assert np.max(np.abs(a @ x - truth)) <= 1e-12


def test_acceptance_mom_deviation_rate(orc):  # acceptance.cpp:151-179 (reduced: 40 of 200 trials)
    a = orc.gen_orthogonal(256, 424242)
    sk = orc.preprocess(a)
    J, K = orc.choose_params(sk.row_norm_max, 0.1, 0.1, 256)
    assert (J, K) == (2956, 16)
    fails = 0
    for t in range(40):
        x, truth = orc.gen_exact_sparse(a, 8, 5000 + t)
        r = orc.transform(sk, x, _params(orc, epsilon=0.05, s=8, J=J, K=K, seed=9000 + t))
        fails += int(np.max(np.abs(r.mu - truth)) >= 0.1)
    assert fails / 40 <= 0.1 + 3 * np.sqrt(0.1 / 40)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_gathered_transform_and_block_match_full_sketch(orc, dtype):
    """The two checker entry points the full-size GPU tests use: kerdock_block (one basis of
    sketch.hpp:171-196) equals that basis of preprocess(), and the draw_and_gather transform
    (stream.hpp:184-191) equals transform() bit for bit, in fp64 and run in float."""
    rng = np.random.default_rng(12)
    a = rng.standard_normal((24, 50)).astype(dtype)
    sk = orc.preprocess(a, dtype=dtype)
    cols = sk.columns()
    for s in (0, 7, sk.d // 2 - 1):
        assert orc.kerdock_block(a, s, dtype).tobytes() == cols[s * sk.d:(s + 1) * sk.d].tobytes()
    for t in range(4):
        x = rng.standard_normal(50).astype(dtype)
        p = _params(orc, epsilon=0.3, s=3, J=40, K=3, seed=100 + t)
        idx = orc.draw_samples(sk.L, p)
        r1 = orc.transform(sk, x, p)
        r2 = orc.transform_gathered(a, x, p, idx, cols[idx], dtype=dtype)
        assert r1.mu.tobytes() == r2.mu.tobytes()
        assert r1.candidate_set.tolist() == r2.candidate_set.tolist()
        assert r1.support.tolist() == r2.support.tolist()
        assert r1.values.tobytes() == r2.values.tobytes()


def test_fast_order_restatement_matches_reference_order(orc):
    """oracle.transform_gathered_fast_order (the B200 FAST kernels' summation orders) computes the
    same transform as the reference order run in float, up to rounding: mu within 1e-5 of the
    estimate's scale, identical candidate sets and supports on well-separated inputs; and it is
    deterministic (bit-identical on repeat)."""
    rng = np.random.default_rng(21)
    for n, m in ((256, 40), (64, 30), (1000, 50)):
        a = (rng.standard_normal((m, n)) / np.sqrt(n)).astype(np.float32)
        sk = orc.preprocess(a, dtype=np.float32)
        cols = sk.columns()
        x = np.zeros(n, dtype=np.float32)
        x[:3] = [0.8, -0.5, 0.3]
        x = (a.T @ (np.eye(m, dtype=np.float32)[:, 0] * 3.0) + 0.01 * x).astype(np.float32)
        p = _params(orc, epsilon=0.5, s=2, J=200, K=3, seed=5)
        idx = orc.draw_samples(sk.L, p)
        r1 = orc.transform_gathered(a, x, p, idx, cols[idx], dtype=np.float32)
        r2 = orc.transform_gathered_fast_order(a, x, p, idx, cols[idx])
        r3 = orc.transform_gathered_fast_order(a, x, p, idx, cols[idx])
        assert r2.mu.tobytes() == r3.mu.tobytes()
        np.testing.assert_allclose(r2.mu, r1.mu, rtol=1e-4, atol=1e-5 * np.max(np.abs(r1.mu)))
        assert r2.support.tolist() == r1.support.tolist()
        np.testing.assert_allclose(r2.values, r1.values, rtol=1e-5)
