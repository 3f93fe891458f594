"""N > 1 host logic on CPU with the gloo backend, world_size 2 (127.0.0.1).

Covers: vector sharding (per-vector seeds independent of the rank split), the
A broadcast, the in-place all-gather of basis-sharded sketch blocks (with a
fake sketch filled from the oracle's per-basis columns), and the
max-over-ranks step time."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2105_05879_b200 import parallel


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, tmpdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as orc
        from paper_2105_05879_b200 import generators
        out = {}
        # --- A broadcast: rank 0 owns the matrix ---
        n, m = 16, 12
        a = torch.from_numpy(np.random.default_rng(7).standard_normal((m, n))) if rank == 0 else \
            torch.zeros((m, n), dtype=torch.float64)
        parallel.broadcast_matrix(a, src=0)
        out["a"] = a.numpy().copy()
        # --- vector shard + seed schedule ---
        first, count = parallel.vector_shard(rank, world, 5)
        g, st = generators.trial_seeds(99, first, count)
        out["seeds"] = st.copy()
        # --- basis-sharded sketch, in-place all-gather ---
        ref = orc.preprocess(out["a"])
        d, L, nk, ldc = ref.d, ref.L, ref.d // 2, ref.m
        full = torch.zeros(L * ldc, dtype=torch.float64)
        b0, cnt = parallel.basis_shards(nk, world)[rank]
        lo, hi = parallel.shard_element_range((b0, cnt), d, ldc)
        full[lo:hi] = torch.from_numpy(ref.columns().reshape(-1)[lo:hi].copy())
        full[nk * d * ldc:] = torch.from_numpy(ref.columns().reshape(-1)[nk * d * ldc:].copy())  # identity: local
        parallel.allgather_basis_shards(full, world, rank, nk, d, ldc)
        out["sketch_ok"] = bool(np.array_equal(full.numpy(), ref.columns().reshape(-1)))
        # --- max over ranks ---
        out["tmax"] = parallel.max_over_ranks(1.5 + rank)
        np.save(os.path.join(tmpdir, f"r{rank}.npy"), out, allow_pickle=True)
    finally:
        dist.destroy_process_group()


def _uneven_worker(rank, world, port, tmpdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as orc
        a = np.random.default_rng(3).standard_normal((5, 16))
        ref = orc.preprocess(a)
        d, L, nk, ldc = ref.d, ref.L, ref.d // 2, ref.m          # nk = 8 bases over 3 ranks: 3 + 3 + 2
        cols = ref.columns().reshape(-1)
        full = torch.zeros(L * ldc, dtype=torch.float64)
        lo, hi = parallel.shard_element_range(parallel.basis_shards(nk, world)[rank], d, ldc)
        full[lo:hi] = torch.from_numpy(cols[lo:hi].copy())
        full[nk * d * ldc:] = torch.from_numpy(cols[nk * d * ldc:].copy())
        parallel.allgather_basis_shards(full, world, rank, nk, d, ldc)
        np.save(os.path.join(tmpdir, f"u{rank}.npy"), np.array([np.array_equal(full.numpy(), cols)]))
    finally:
        dist.destroy_process_group()


def test_three_rank_uneven_basis_allgather(tmp_path):
    """World sizes that do not divide the basis count: per-rank broadcasts."""
    world, port = 3, _free_port()
    mp.spawn(_uneven_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert np.load(tmp_path / f"u{r}.npy")[0]


def test_two_rank_gloo(tmp_path):
    world, port = 2, _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    r0 = np.load(tmp_path / "r0.npy", allow_pickle=True).item()
    r1 = np.load(tmp_path / "r1.npy", allow_pickle=True).item()
    assert np.array_equal(r0["a"], r1["a"])
    assert r0["sketch_ok"] and r1["sketch_ok"]
    assert r0["tmax"] == r1["tmax"] == 2.5
    # the per-vector seeds of ranks 0 and 1 are exactly the single-process schedule
    from paper_2105_05879_b200 import generators
    _, allseeds = generators.trial_seeds(99, 0, 10)
    assert np.array_equal(np.concatenate([r0["seeds"], r1["seeds"]]), allseeds)


def test_shard_plans():
    for nk, world in [(2048, 8), (2048, 3), (129, 8), (8, 8), (1, 4)]:
        shards = parallel.basis_shards(nk, world)
        covered = []
        for first, count in shards:
            covered += list(range(first, first + count))
        assert covered == list(range(nk))
        sizes = [c for _, c in shards]
        assert max(sizes) - min(sizes) <= 1
    assert parallel.vector_shard(3, 8, 65536) == (3 * 65536, 65536)
    with pytest.raises(ValueError):
        parallel.vector_shard(8, 8, 1)
    assert parallel.shard_element_range((256, 256), 4096, 4096) == (256 * 4096 * 4096, 512 * 4096 * 4096)


def _route_worker(rank, world, port, tmpdir):
    """Config-4 routing (parallel.RoutingPlan / route_retained_columns) on gloo:
    each rank computes only the columns of its basis shard (oracle columns
    A s_ell), the all-to-all delivers them, and every rank's gathered buffer
    must equal the direct draw_and_gather of its own vectors."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as orc
        k, n, m = 4, 13, 11
        d, nk = 1 << k, (1 << k) // 2
        L = d * (nk + 1)
        a = np.random.default_rng(3).standard_normal((m, n))
        ok = []
        for B, N in [(5, 7), (1, 3), (9, 40)]:
            idx_all = np.random.default_rng(B * 100 + N).integers(0, L, size=(B, N))
            idx_all[0, 0] = L - 1                                   # identity block -> last rank
            vec_ranges = [parallel.strong_shard(q, world, B) for q in range(world)]
            shards = parallel.basis_shards(nk, world)
            plan = parallel.RoutingPlan(idx_all, vec_ranges, shards, d, nk, rank)
            computed = []

            def sample_fn(ells):
                owners = parallel.column_owner(ells, shards, d, nk)
                assert np.all(owners == rank)                       # only my basis shard is computed here
                computed.append(len(ells))
                return torch.from_numpy(orc.design_columns(k, n, ells) @ a.T)

            got = parallel.route_retained_columns(plan, sample_fn, m, torch.float64, "cpu")
            first, count = vec_ranges[rank]
            want = orc.design_columns(k, n, idx_all[first:first + count].ravel()) @ a.T if count else np.zeros((0, m))
            ok.append(bool(got.shape == (count * N, m) and np.array_equal(got.numpy(), want)))
        np.save(os.path.join(tmpdir, f"route{rank}.npy"), {"ok": ok}, allow_pickle=True)
    finally:
        dist.destroy_process_group()


def test_two_rank_config4_routing(tmp_path):
    world, port = 2, _free_port()
    mp.spawn(_route_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert all(np.load(tmp_path / f"route{r}.npy", allow_pickle=True).item()["ok"])


def test_routing_plan_single_process():
    """Plan bookkeeping for 3 ranks without a process group: every (vector, sample)
    is sent exactly once, by the owner of its basis, to the owner of its vector."""
    d, nk, L = 16, 8, 16 * 9
    rng = np.random.default_rng(5)
    idx_all = rng.integers(0, L, size=(10, 6))
    vec_ranges = [parallel.strong_shard(q, 3, 10) for q in range(3)]
    shards = parallel.basis_shards(nk, 3)
    plans = [parallel.RoutingPlan(idx_all, vec_ranges, shards, d, nk, r) for r in range(3)]
    N = idx_all.shape[1]
    for q in range(3):                                   # what q receives from r == what r sends to q
        for r in range(3):
            assert plans[q].recv_counts[r] == plans[r].send_counts[q]
        assert plans[q].recv_counts.sum() == vec_ranges[q][1] * N
        assert sorted(plans[q].recv_positions.tolist()) == list(range(vec_ranges[q][1] * N))
    assert sum(len(p.send_ells) for p in plans) == idx_all.size
    assert parallel.column_owner(np.array([L - 1]), shards, d, nk)[0] == 2
    assert parallel.column_owner(np.array([0]), parallel.basis_shards(1, 4), d, 1)[0] == 0
    with pytest.raises(ValueError):
        parallel.RoutingPlan(idx_all, vec_ranges[:2], shards, d, nk, 0)


def _means_worker(rank, world, port, tmpdir):
    """Config-4 row-sharded routing: each rank holds the batch means of its row
    shard for every vector; after route_partial_means every rank holds the
    complete means of its own vectors."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ok = []
        for B, m, K in [(5, 10, 2), (7, 33, 3), (2, 8, 1)]:
            M = torch.from_numpy(np.random.default_rng(B * m + K).standard_normal((B, K, m)))
            vec_ranges = [parallel.strong_shard(q, world, B) for q in range(world)]
            row_ranges = [(f, f + c) for f, c in (parallel.strong_shard(r, world, m) for r in range(world))]
            r0, r1 = row_ranges[rank]
            ld = (m + 3) // 4 * 4
            full = parallel.route_partial_means(M[:, :, r0:r1].contiguous(), vec_ranges, row_ranges, rank, ld)
            first, count = vec_ranges[rank]
            ok.append(bool(full.shape == (count, K + 1, ld) and torch.equal(full[:, :K, :m], M[first:first + count])))
        np.save(os.path.join(tmpdir, f"means{rank}.npy"), {"ok": ok}, allow_pickle=True)
    finally:
        dist.destroy_process_group()


def test_two_rank_row_sharded_means(tmp_path):
    world, port = 2, _free_port()
    mp.spawn(_means_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert all(np.load(tmp_path / f"means{r}.npy", allow_pickle=True).item()["ok"])
