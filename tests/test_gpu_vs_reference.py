"""GPU path against the REFERENCE ITSELF (not the restatement).

oracle/_ref/libfst_ref.so is the reference's own sketch.hpp / stream.hpp code compiled
from its sources against the Eigen-API shim (tests/test_ref_pin.py pins it to the
oracle on the CPU). Here the sm_100a library runs through its C-ABI and is compared
with that build on the same inputs, in fp64 STRICT mode where north_star asks for
identical supports and values within 1e-12:
  * n = 256 (config-1 shape): every sketch column bit-identical to the reference's
    preprocess(); B = 300 (persistent non-split kernel) and B = 5 (batch-split path):
    every vector's mu, candidate set and support bit-identical, values within 1e-12;
  * n = 1024 iid A (config-2 shape, fp64): B = 400, every vector.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fst():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from oracle import refimpl
    if not refimpl.available():
        pytest.skip("oracle/_ref/libfst_ref.so not built")
    from paper_2105_05879_b200 import fst
    return fst


def _check_batch(fst, ref, rsk, sk, X, seeds, eps, s, J, K):
    from oracle import oracle as orc
    p = fst.StreamParams(epsilon=eps, s=s, J=J, K=K, mode=fst.MODE_STRICT)
    out = fst.transform_batch(sk, X, p, seeds=seeds, candidates=True, mu=True)
    for v in range(X.shape[0]):
        r = ref.transform(rsk, X[v], orc.StreamParams(epsilon=eps, s=s, J=J, K=K, seed=int(seeds[v])))
        g = out.result(v)
        assert g.mu.tobytes() == r.mu.tobytes(), v
        assert g.candidate_set.tolist() == r.candidate_set.tolist(), v
        assert g.support.tolist() == r.support.tolist(), v
        np.testing.assert_allclose(g.values, r.values, rtol=1e-12, atol=1e-15)


def test_config1_shape_sketch_and_transform_vs_reference(fst):
    from oracle import oracle as orc
    from oracle import refimpl as ref
    n = 256
    a = orc.gen_orthogonal(n, 777)
    rsk = ref.preprocess(a, threads=os.cpu_count() or 1)
    sk = fst.preprocess(a, device=0)
    cols = np.stack([sk.column(ell) for ell in range(sk.L)])
    assert cols.tobytes() == rsk.columns().tobytes()
    for B in (300, 5):
        X = np.stack([orc.gen_exact_sparse(a, 8, orc.gen_seed(9000 + v))[0] for v in range(B)])
        seeds = np.array([orc.stream_seed(9000 + v) for v in range(B)], dtype=np.uint64)
        _check_batch(fst, ref, rsk, sk, X, seeds, 0.1, 8, 375, 2)
    sk.close()


def test_config2_shape_fp64_vs_reference(fst):
    from oracle import oracle as orc
    from oracle import refimpl as ref
    n, B = 1024, 400
    g = orc.rng_gaussian(1024, n * n).reshape(n, n) / np.sqrt(n)
    rsk = ref.preprocess(g, threads=os.cpu_count() or 1)
    sk = fst.preprocess(g, device=0)
    rng = np.random.default_rng(23)
    X = rng.standard_normal((B, n))
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    seeds = np.array([orc.stream_seed(11000 + v) for v in range(B)], dtype=np.uint64)
    _check_batch(fst, ref, rsk, sk, X, seeds, 0.05, 16, 375, 2)
    sk.close()
