"""GPU experiment harness vs the reference harness semantics (experiment.hpp):
config parsing (CPU), generator parity with gen_mixture / gen_exact_sparse
(CPU), and per-grid-point errors equal to the oracle's per-trial loop (GPU)."""
import numpy as np
import pytest

from paper_2105_05879_b200 import experiment, generators


def test_parse_config_and_csv():
    cfg = experiment.parse_config("n = 64\ns = 4 # comment\ntrials = 10\nJgrid = 20,50\nKgrid = 2,3\n"
                                  "epsilon = 0.25\nseed = 99\nmode = exact-sparse\n")
    assert (cfg.n, cfg.s, cfg.trials, cfg.j_grid, cfg.k_grid, cfg.epsilon, cfg.seed) == \
        (64, 4, 10, [20, 50], [2, 3], 0.25, 99)
    with pytest.raises(ValueError):
        experiment.parse_config("bogus = 1")
    with pytest.raises(ValueError):
        experiment.parse_config("mode = other")
    with pytest.raises(ValueError):
        experiment.parse_config("n 4")
    csv = experiment.to_csv([experiment.ExperimentRow(20, 2, 0.5, 0.0, 0.25)])
    assert csv.splitlines() == ["J,K,worst_inf_err,worst_l2_err,runtime_ratio", "20,2,0.5,0,0.25"]


def test_target_generators_match_reference_draws(orc):
    a = orc.gen_orthogonal(32, 5)
    for seed in [1, 77, 2**63 + 3]:
        _, truth = orc.gen_exact_sparse(a, 4, seed)
        y = generators.sparse_targets(np.array([seed], dtype=np.uint64), 32, 4)[0]
        assert np.array_equal(y, truth)
        x, truth = orc.gen_mixture(a, 0.2, seed)
        import ctypes as C
        from paper_2105_05879_b200 import fst
        ym = np.zeros(32)
        s = np.array([seed], dtype=np.uint64)
        fst._check(fst.lib().fstg_gen_mixture_targets(s.ctypes.data_as(C.c_void_p), 1, 32, C.c_double(0.2),
                                                       ym.ctypes.data_as(C.c_void_p)))
        xr = a.T @ ym
        np.testing.assert_allclose(ym / np.linalg.norm(xr), truth, rtol=1e-12, atol=1e-15)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["exact-sparse", "gaussian-mixture"])
def test_run_experiment_matches_oracle_loop(orc, mode):
    import torch
    from paper_2105_05879_b200 import fst
    n = 64
    a = orc.gen_orthogonal(n, 777)
    A64 = torch.from_numpy(a).cuda()
    sk = fst.preprocess(a)  # fp64: STRICT arithmetic, mu bit-exact
    cfg = experiment.ExperimentConfig(n=n, s=4, trials=12, j_grid=[20, 50], k_grid=[2, 3], epsilon=0.25,
                                      seed=99, mode=mode, mixture_p=0.1)
    rows = experiment.run_experiment(cfg, sk, A64)
    ref = orc.preprocess(a)
    X64, seeds = experiment.trial_inputs(A64, cfg)
    X = X64.cpu().numpy()
    for row in rows:
        inf_err = l2_err = 0.0
        for t in range(cfg.trials):
            r = orc.transform(ref, X[t], orc.StreamParams(epsilon=0.25, s=4, J=row.J, K=row.K, seed=int(seeds[t])))
            ax = a @ X[t]
            inf_err = max(inf_err, np.max(np.abs(r.mu - ax)))
            h = np.zeros(n)
            h[r.support] = r.values
            l2_err = max(l2_err, np.linalg.norm(h - orc.hard_threshold(ax, 0.25)))
        assert row.worst_inf_err == pytest.approx(inf_err, rel=1e-9, abs=1e-12)
        assert row.worst_l2_err == pytest.approx(l2_err, rel=1e-9, abs=1e-12)
        assert row.runtime_ratio > 0
