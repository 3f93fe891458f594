"""Properties the reference's own suites check, on the GPU path (test_sketch.cpp
/ test_stream.cpp names cited per test): design-level identities, linearity,
determinism and concurrent use of one shared sketch. GPU."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fst():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2105_05879_b200 import fst
    return fst


def test_identity_matrix_reproduces_design_columns(fst, orc):
    """test_sketch.cpp 'preprocess of the identity reproduces the design columns':
    column ell of preprocess(I_n) is the projected design vector s_ell."""
    for n in (16, 13, 64):
        sk = fst.preprocess(np.eye(n))
        ells = np.arange(sk.L, dtype=np.int64)
        want = orc.design_columns(sk.k, n, ells)                      # (L, n)
        got = fst.sample_columns(sk, ells)[:, :n]
        assert np.array_equal(got, want)


def test_all_ones_row(fst):
    """test_sketch.cpp 'single all-ones row: Kerdock(0,0) column sums the row' (Q_0 = 0, w = 0)."""
    for n in (16, 50, 256):
        a = np.random.default_rng(n).standard_normal((1, n))
        sk = fst.preprocess(a)
        assert sk.column(0)[0] == pytest.approx(a.sum(), rel=1e-12)
        ones = fst.preprocess(np.ones((1, n)))
        assert ones.column(0)[0] == float(n)


def test_mean_identity_over_the_whole_design(fst, orc):
    """test_sketch.cpp 'mean identity' / test_stream.cpp 'estimator is unbiased over a
    deterministic sweep of the design': with every design index as a sample
    (J = L, K = 1) the estimate (1/L) sum_ell t_ell C[:, ell] is exactly Ax."""
    for n, m in ((16, 16), (16, 9), (64, 40)):
        a = np.random.default_rng(n + m).standard_normal((m, n))
        x = np.random.default_rng(n * m).standard_normal(n)
        sk = fst.preprocess(a)
        p = fst.StreamParams(epsilon=1e-9, s=m, J=sk.L, K=1)     # fp64: STRICT by default
        r = fst.transform_with_samples(sk, x, p, np.arange(sk.L, dtype=np.int64))
        np.testing.assert_allclose(r.mu, a @ x, rtol=1e-12, atol=1e-12)


def test_preprocess_is_linear(fst):
    """test_sketch.cpp 'preprocess scales linearly in A': scaling by 2 is exact in
    floating point, sums agree to rounding."""
    rng = np.random.default_rng(3)
    a, b = rng.standard_normal((20, 100)), rng.standard_normal((20, 100))
    ells = rng.integers(0, fst.preprocess(a).L, size=200)
    ca = fst.sample_columns(fst.preprocess(a), ells)
    c2a = fst.sample_columns(fst.preprocess(2.0 * a), ells)
    cab = fst.sample_columns(fst.preprocess(a + b), ells)
    cb = fst.sample_columns(fst.preprocess(b), ells)
    assert np.array_equal(c2a, 2.0 * ca)
    np.testing.assert_allclose(cab, ca + cb, rtol=1e-12, atol=1e-11)


def test_builds_and_transforms_are_deterministic(fst):
    """test_sketch.cpp 'sketch build is identical across thread counts' and
    test_stream.cpp 'transform is deterministic': repeated builds / runs are bitwise equal."""
    a = np.random.default_rng(9).standard_normal((300, 1000)).astype(np.float32)
    s1, s2 = fst.preprocess(a), fst.preprocess(a)
    ells = np.random.default_rng(1).integers(0, s1.L, size=500)
    assert fst.sample_columns(s1, ells).tobytes() == fst.sample_columns(s2, ells).tobytes()
    X = np.random.default_rng(2).standard_normal((50, 1000)).astype(np.float32)
    p = fst.StreamParams(epsilon=0.5, s=4, J=30, K=3)
    seeds = np.arange(50, dtype=np.uint64)
    r1 = fst.transform_batch(s1, X, p, seeds=seeds, mu=True)
    r2 = fst.transform_batch(s2, X, p, seeds=seeds, mu=True)
    assert np.array_equal(r1.counts, r2.counts) and r1.mu.tobytes() == r2.mu.tobytes()
    s1.close()
    s2.close()


def test_concurrent_transforms_on_one_sketch(fst):
    """test_stream.cpp 'concurrent transforms over one shared sketch agree with serial
    runs': four host threads, each on its own CUDA stream, share one sketch."""
    import torch
    a = np.random.default_rng(4).standard_normal((128, 256)).astype(np.float32)
    sk = fst.preprocess(a)
    p = fst.StreamParams(epsilon=0.5, s=4, J=40, K=2)
    Xs = [np.random.default_rng(10 + t).standard_normal((300, 256)).astype(np.float32) for t in range(4)]
    seeds = [np.arange(300, dtype=np.uint64) + 1000 * t for t in range(4)]
    serial = [fst.transform_batch(sk, Xs[t], p, seeds=seeds[t], mu=True) for t in range(4)]
    results, errors = [None] * 4, []

    def work(t):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                for _ in range(3):
                    results[t] = fst.transform_batch(sk, Xs[t], p, seeds=seeds[t], mu=True, stream=st.cuda_stream)
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    threads = [threading.Thread(target=work, args=(t,)) for t in range(4)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors
    for t in range(4):
        assert np.array_equal(results[t].counts, serial[t].counts)
        valid = np.arange(serial[t].support.shape[1])[None, :] < serial[t].counts[:, None]
        assert np.array_equal(results[t].support[valid], serial[t].support[valid])
        assert np.array_equal(results[t].values[valid], serial[t].values[valid])
        assert results[t].mu.tobytes() == serial[t].mu.tobytes()
    sk.close()


def test_public_helpers_match_oracle(fst, orc):
    """inner_product_with_design (bit-exact Gray-code walk), median_of_means,
    hard_threshold and projected_design_column on the GPU vs the oracle
    (test_stream.cpp 'inner_product_with_design fixed values / matches the
    materialized oracle', 'median_of_means fixed values', 'hard_threshold ...')."""
    rng = np.random.default_rng(12)
    for k, n in ((2, 4), (4, 13), (6, 64), (8, 200), (12, 4096)):
        d = 1 << k
        L = d * (d // 2 + 1)
        x = rng.standard_normal(n)
        for ell in list(rng.integers(0, L, size=20)) + [0, L - 1, L - d, d * (d // 2) - 1]:
            g = fst.inner_product_with_design(x, k, int(ell))
            assert g == orc.inner_product_with_design(x, k, int(ell)), (k, ell)
            col = fst.projected_design_column(k, n, int(ell))
            assert np.array_equal(col, orc.projected_design_column(k, n, int(ell)))
    for m, J, K in ((7, 5, 1), (9, 4, 2), (16, 3, 5), (33, 2, 4)):
        smp = rng.standard_normal((m, J * K))
        np.testing.assert_allclose(fst.median_of_means(smp, J, K), orc.median_of_means(smp, J, K), rtol=1e-12,
                                   atol=1e-15)
    v = np.array([0.5, -0.1, 0.1, 0.09999, -0.2, 0.0])
    assert np.array_equal(fst.hard_threshold(v, 0.1), orc.hard_threshold(v, 0.1))
    with pytest.raises(ValueError):
        fst.inner_product_with_design(np.zeros(17), 4, 0)
    with pytest.raises(IndexError):
        fst.projected_design_column(4, 16, 16 * 9)
    with pytest.raises(ValueError):
        fst.median_of_means(np.zeros((3, 5)), 2, 2)


def test_embedded_matrix(fst, tmp_path):
    """sketch.hpp:107-111: the embedded A round-trips; a sketch loaded without A raises."""
    a = np.random.default_rng(3).standard_normal((7, 13))
    sk = fst.preprocess(a)
    assert np.array_equal(sk.embedded_matrix(), a)
    des = fst.preprocess_design(a.astype(np.float32))
    assert np.array_equal(des.embedded_matrix(), a.astype(np.float32))


def test_size_limits_fail_loudly(fst):
    """Largest supported column height (m = 16384 fp32, four 16 KiB segments) works;
    one row more is rejected with NotSupportedError (no silent fallback)."""
    import torch
    p = fst.StreamParams(epsilon=0.5, s=1, J=3, K=2)
    for m, ok in ((16384, True), (16385, False)):
        a = torch.randn(m, 8, device="cuda:0", generator=torch.Generator("cuda:0").manual_seed(m))
        sk = fst.preprocess(a)
        X = torch.randn(2, 8, device="cuda:0")
        if ok:
            out = fst.transform_batch(sk, X, p, seeds=np.arange(2, dtype=np.uint64))
            assert int(out.counts.max()) >= 0
        else:
            with pytest.raises(fst.NotSupportedError):
                fst.transform_batch(sk, X, p, seeds=np.arange(2, dtype=np.uint64))
        sk.close()


@pytest.mark.parametrize("dtype,mode,K", [(np.float32, 0, 2), (np.float64, 0, 16), (np.float32, 2, 3)])
def test_small_batch_split_equals_large_batch(fst, dtype, mode, K):
    """Batches smaller than the SM count run one (vector, batch) pair per work item,
    then the tail from the batch means. Every output equals the same vectors run
    inside a large (unsplit) batch, bit for bit."""
    rng = np.random.default_rng(K)
    a = rng.standard_normal((200, 256)).astype(dtype)
    sk = fst.preprocess(a)
    p = fst.StreamParams(epsilon=0.5, s=3, J=37, K=K, mode=mode)
    X = rng.standard_normal((300, 256)).astype(dtype)
    seeds = rng.integers(0, 2**63, size=300, dtype=np.int64).view(np.uint64)
    big = fst.transform_batch(sk, X, p, seeds=seeds, candidates=True, mu=True)      # 300 >= #SMs: unsplit
    small = fst.transform_batch(sk, X[:5], p, seeds=seeds[:5], candidates=True, mu=True)  # split
    assert np.array_equal(big.counts[:5], small.counts)
    valid = np.arange(small.support.shape[1])[None, :] < small.counts[:, None]
    assert np.array_equal(big.support[:5][valid], small.support[valid])
    assert np.array_equal(big.values[:5][valid], small.values[valid])
    assert np.array_equal(big.candidates[:5], small.candidates)
    assert big.mu[:5].tobytes() == small.mu.tobytes()
    sk.close()
