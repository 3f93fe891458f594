"""Design verifiers (kerdock.hpp:198-317, cli.hpp:45-60).

CPU: the oracle restatement against the reference's own known answers
(test_kerdock.cpp:200-256, acceptance.cpp:31-66). GPU: fstg_verify_* under the
reference policy must reproduce the oracle's reports exactly (every value is
an exact dyadic rational), and the exhaustive policy checks every basis pair
up to k = 14 (the config-4 design)."""
import time

import numpy as np
import pytest


# ------------------------------------------------------------------ oracle ----
@pytest.mark.parametrize("k", [2, 4])
def test_oracle_mub_exact_small_k(orc, k):  # test_kerdock.cpp:200-211
    rep = orc.verify_mub(k)
    inv_d = 1.0 / (1 << k)
    assert rep.exhaustive
    assert rep.max_within_gram_dev <= 1e-12
    assert rep.min_cross_sq == pytest.approx(inv_d, rel=1e-12)
    assert rep.max_cross_sq == pytest.approx(inv_d, rel=1e-12)


def test_oracle_mub_cap(orc):  # test_kerdock.cpp:213-216
    with pytest.raises(ValueError):
        orc.verify_mub(6, cap=4)
    with pytest.raises(ValueError):
        orc.verify_design_moments(6, cap=4)


def test_oracle_mub_structure_k6(orc):  # acceptance.cpp:53-62
    rep = orc.verify_mub(6)
    assert rep.exhaustive and rep.max_within_gram_dev <= 1e-10 and rep.max_cross_dev <= 1e-10


def test_oracle_k8_sampled(orc):  # test_kerdock.cpp:218-229
    mub = orc.verify_mub(8)
    assert not mub.exhaustive
    assert mub.max_within_gram_dev <= 1e-10 and mub.max_cross_dev <= 1e-10
    rep = orc.verify_design_moments(8)
    assert not rep.exact
    assert rep.m1 == pytest.approx(orc.design_moment_target(256, 1), rel=0.05)
    assert abs(rep.m2 - orc.design_moment_target(256, 2)) <= 1e-4


def test_oracle_moments_match_targets(orc):  # test_kerdock.cpp:231-247, acceptance.cpp:31-51
    rep = orc.verify_design_moments(2)
    assert rep.exact and rep.m1 == pytest.approx(0.25, rel=1e-12) and rep.m2 == pytest.approx(0.125, rel=1e-12)
    rep = orc.verify_design_moments(4)
    assert rep.m1 == pytest.approx(1 / 16, rel=1e-12) and rep.m2 == pytest.approx(1 / 96, rel=1e-12)
    assert orc.design_moment_target(16, 1) == pytest.approx(1 / 16)
    assert orc.design_moment_target(16, 2) == pytest.approx(1 / 96)
    rep = orc.verify_design_moments(6)
    assert abs(rep.m1 - 1 / 64) <= 1e-9 and abs(rep.m2 - 3 / (64 * 66)) <= 1e-9


def test_oracle_single_basis_is_flagged(orc):  # test_kerdock.cpp:250-257
    rep = orc.design_moments_of(np.eye(16))
    assert rep.m1 == pytest.approx(1 / 16) and rep.m2 == pytest.approx(1 / 16)
    assert abs(rep.m2 - orc.design_moment_target(16, 2)) > 1e-3


@pytest.mark.parametrize("k", [2, 4, 6, 8])
def test_oracle_kerdock_property(orc, k):  # acceptance.cpp:64-75, cli.hpp:45-60
    skew, bad = orc.verify_kerdock_set(k)
    assert skew and bad == 0


def test_moment_target_host_function(orc):
    from paper_2105_05879_b200 import fst
    for d in (4, 16, 64, 256, 4096, 16384):
        for j in (1, 2, 3):
            assert fst.design_moment_target(d, j) == orc.design_moment_target(d, j)


# ------------------------------------------------------------------- GPU ----
@pytest.fixture(scope="module")
def fst():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2105_05879_b200 import fst
    return fst


@pytest.mark.gpu
@pytest.mark.parametrize("k", [2, 4, 6, 8])
def test_gpu_reference_policy_equals_oracle(fst, orc, k):
    g, o = fst.verify_mub(k), orc.verify_mub(k)
    assert (g.max_within_gram_dev, g.min_cross_sq, g.max_cross_sq, g.max_cross_dev, g.exhaustive) == tuple(o)
    gm, om = fst.verify_design_moments(k), orc.verify_design_moments(k)
    assert (gm.m1, gm.m2, gm.exact) == tuple(om), (gm, om)


@pytest.mark.gpu
def test_gpu_cap_and_errors(fst):
    with pytest.raises(ValueError):
        fst.verify_mub(6, cap=4)
    with pytest.raises(ValueError):
        fst.verify_design_moments(6, cap=4)
    with pytest.raises(ValueError):
        fst.verify_mub(5)                      # odd k (DesignParams::make)
    with pytest.raises(ValueError):
        fst.verify_mub(4, policy=7)


@pytest.mark.gpu
@pytest.mark.parametrize("k", [8, 10, 12, 14])
def test_gpu_exhaustive_mub_and_moments(fst, k):
    d = 1 << k
    nb = d // 2 + 1
    t0 = time.perf_counter()
    rep = fst.verify_mub(k, cap=14, policy=fst.VERIFY_EXHAUSTIVE)
    t1 = time.perf_counter()
    assert rep.exhaustive and rep.basis_pairs == nb * (nb - 1) // 2
    assert rep.max_within_gram_dev == 0.0 and rep.max_cross_dev == 0.0
    assert rep.min_cross_sq == rep.max_cross_sq == 1.0 / d
    mom = fst.verify_design_moments(k, cap=14, policy=fst.VERIFY_EXHAUSTIVE)
    t2 = time.perf_counter()
    assert mom.exact and mom.pairs == (nb * d) ** 2
    assert mom.m1 == fst.design_moment_target(d, 1)
    assert mom.m2 == pytest.approx(fst.design_moment_target(d, 2), rel=1e-15)
    print(f"k={k}: exhaustive MUB {t1 - t0:.3f} s, moments {t2 - t1:.3f} s")


@pytest.mark.gpu
@pytest.mark.parametrize("k", [2, 4, 6, 8, 10])
def test_gpu_kerdock_set_matches_oracle(fst, orc, k):
    assert fst.verify_kerdock_set(k) == orc.verify_kerdock_set(k) == (True, 0)


@pytest.mark.gpu
def test_gpu_kerdock_set_k14(fst):
    t0 = time.perf_counter()
    assert fst.verify_kerdock_set(14) == (True, 0)   # 33.5M basis pairs, all full rank
    print(f"k=14 rank check {time.perf_counter() - t0:.3f} s")
