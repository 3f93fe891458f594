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
