"""Parity on the other BASELINE configurations (config 3 is covered in
test_gpu_parity.py): config 2 (iid A, x = A^-1 y, eps = 0.05, s = 16) and
config 5's large candidate sets (n = 4096, s = 64 / 256 -> want = 640 / 2560)
against the oracle's draw_and_gather path (stream.hpp:184-191, 197-268) on the
GPU's own gathered columns (the columns themselves are pinned bit-exact in
test_gpu_parity.py). GPU."""
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


def _check_vs_gathered(fst, orc, sk, prob, J, K, nvec):
    """GPU transform of nvec vectors vs the oracle on the same (fp64-widened) columns."""
    import torch
    from test_gpu_parity import _support_diff_allowed
    want = fst.candidate_count(prob.s, 10, sk.m)
    p = fst.StreamParams(epsilon=prob.eps, s=prob.s, J=J, K=K)
    seeds = prob.seeds[:nvec]
    out = fst.transform_batch(sk, prob.X[:nvec].contiguous(), p,
                              seeds=torch.as_tensor(seeds.astype(np.int64)).cuda(), candidates=True, mu=True)
    idx = fst.draw_samples(sk, p, seeds=seeds)
    a64 = prob.A.double().cpu().numpy()
    X = prob.X[:nvec].double().cpu().numpy()
    supports = []
    for v in range(nvec):
        gathered = fst.sample_columns(sk, idx[v])[:, :sk.m].astype(np.float64)
        r = orc.transform_gathered(a64, X[v], orc.StreamParams(epsilon=prob.eps, s=prob.s, J=J, K=K), idx[v],
                                   gathered)
        g = out.result(v)
        np.testing.assert_allclose(g.mu, r.mu, rtol=1e-4, atol=5e-6)
        assert _support_diff_allowed(g, r, r.mu, a64 @ X[v], prob.eps, want)
        common = sorted(set(g.support.tolist()) & set(r.support.tolist()))
        gi = {i: k for k, i in enumerate(g.support.tolist())}
        ri = {i: k for k, i in enumerate(r.support.tolist())}
        for i in common:
            assert g.values[gi[i]] == pytest.approx(r.values[ri[i]], rel=1e-5)
        supports.append(len(r.support))
    return supports


def test_config2_iid_inverse_targets(fst, orc):
    """Config 2: A iid N(0,1/n), n = 1024, x = A^-1 y / |.|, y 16-sparse N(0,1), eps = 0.05.
    The true support of Ax is (almost always) empty; GPU and oracle agree vector by vector."""
    from paper_2105_05879_b200 import generators
    prob = generators.config2_problem(B=6, seed=20251020, device="cuda:0")
    sk = fst.preprocess(prob.A)
    supports = _check_vs_gathered(fst, orc, sk, prob, 375, 2, 6)
    ax = (prob.A.double() @ prob.X.double().T).abs().cpu().numpy()
    assert int((ax >= prob.eps).sum()) <= 2          # predicted ~empty true support
    assert max(supports) <= 2
    sk.close()


@pytest.mark.parametrize("s,eps", [(64, 0.1), (256, 0.05)])
def test_config5_large_candidate_sets_full_size(fst, orc, s, eps):
    """Config 5 at n = 4096 on the real 137.5 GB sketch: want = 640 / 2560 candidates
    (the TMA refinement ring cycles 107 / 427 times per vector)."""
    from paper_2105_05879_b200 import generators
    prob = generators.config5_problem(s, eps, B=2, seed=20251021, device="cuda:0")
    sk = fst.preprocess(prob.A)
    _check_vs_gathered(fst, orc, sk, prob, 375, 2, 2)
    sk.close()


def test_fp64_strict_bit_exact_at_n1024(fst, orc):
    """The reference's own precision at a larger scale: fp64 STRICT at n = 1024
    (4.3 GB sketch), mu bit-exact, candidate sets and supports identical, values
    within 1e-12, against the oracle on the GPU's gathered fp64 columns."""
    from paper_2105_05879_b200 import generators
    n = 1024
    A64 = generators.iid_gaussian(n, 1024, "cuda:0")
    sk = fst.preprocess(A64)
    rng = np.random.default_rng(7)
    X = rng.standard_normal((3, n))
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    seeds = np.array([101, 202, 303], dtype=np.uint64)
    p = fst.StreamParams(epsilon=0.05, s=16, J=120, K=3)
    out = fst.transform_batch(sk, X, p, seeds=seeds, candidates=True, mu=True)
    idx = fst.draw_samples(sk, p, seeds=seeds)
    a64 = A64.cpu().numpy()
    for v in range(3):
        gathered = fst.sample_columns(sk, idx[v])[:, :n]
        r = orc.transform_gathered(a64, X[v], orc.StreamParams(epsilon=0.05, s=16, J=120, K=3), idx[v], gathered)
        g = out.result(v)
        assert g.mu.tobytes() == r.mu.tobytes()
        assert g.candidate_set.tolist() == r.candidate_set.tolist()
        assert g.support.tolist() == r.support.tolist()
        np.testing.assert_allclose(g.values, r.values, rtol=1e-12)
    sk.close()
