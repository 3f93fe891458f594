"""Input generators: the product library's SeededRng fills and target
generator against the oracle's (bit for bit — this is what gives bench.py's two arms the same
inputs), and haar_orthogonal (torch/cuSOLVER QR with diag(R) > 0) against the oracle's
Householder restatement of gen_orthogonal (generators.hpp:20-33)."""
import numpy as np
import pytest

from paper_2105_05879_b200 import generators


def test_gaussian_fill_matches_oracle(orc):
    for seed in (0, 4096, 2**63 + 11):
        assert generators.gaussian(seed, 5001).tobytes() == orc.rng_gaussian(seed, 5001).tobytes()


@pytest.mark.parametrize("value_kind,noise", [(0, 1e-3), (1, 0.0), (0, 0.0)])
def test_sparse_targets_match_oracle(orc, value_kind, noise):
    g, _ = generators.trial_seeds(20251019, 0, 300)
    a = generators.sparse_targets(g, 4096, 32, value_kind=value_kind, noise_sigma=noise)
    b = orc.gen_sparse_targets(g, 4096, 32, value_kind, noise)
    assert a.tobytes() == b.tobytes()
    assert ((a != 0).sum(axis=1) == (4096 if noise else 32)).all()


def test_sparse_targets_match_gen_exact_sparse(orc):
    """value_kind 0 without noise is gen_exact_sparse's truth vector (generators.hpp:44-53)."""
    a = orc.gen_orthogonal(64, 5)
    for seed in (1, 2, 3):
        _, truth = orc.gen_exact_sparse(a, 8, seed)
        y = generators.sparse_targets(np.array([seed], dtype=np.uint64), 64, 8)[0]
        assert y.tobytes() == truth.tobytes()


def _haar_vs_oracle(orc, n, device):
    q = generators.haar_orthogonal(n, 5150 + n, device).cpu().numpy()
    ref = orc.gen_orthogonal(n, 5150 + n)
    return float(np.max(np.abs(q - ref)))


def test_haar_orthogonal_cpu_matches_gen_orthogonal(orc):
    assert _haar_vs_oracle(orc, 256, "cpu") <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("n", [256, 1024])
def test_haar_orthogonal_gpu_matches_gen_orthogonal(orc, n):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    assert _haar_vs_oracle(orc, n, "cuda:0") <= 1e-12
