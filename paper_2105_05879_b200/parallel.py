"""Multi-GPU plumbing for the thresholded-Ax stream (one process per GPU).

The path shards naturally: every vector is an independent
unit with its own seed, so the stream is split by global vector index with no
data-path collective; the representation is replicated per GPU. The only
collectives are in preparation:

  * ``broadcast_matrix``   — A from rank 0 to every rank (NCCL over NVLink).
  * ``allgather_sketch``   — basis-sharded preprocessing: rank r builds Kerdock
    bases ``basis_shards(nk, world)[r]`` (a contiguous byte range of the
    column-major sketch) and an in-place all-gather over NVLink completes every
    replica (option (ii) of §8(e); option (i), local recompute after the
    broadcast, is the default because it moves 64 MB instead of ~120 GB).
  * ``route_retained_columns`` — config 4 (n = 16384, no sketch can exist,
    §8(e) step 3): rank r computes the sampled columns whose Kerdock basis
    lies in its basis shard (the identity block belongs to the last rank),
    for every vector of the chunk, and one all-to-all sends each column to
    the rank that owns its vector, which scatters them into the
    draw_and_gather layout (stream.hpp:184-191). The O(n^3 log n) Kerdock
    pass splits across ranks, and a chunk can hold world x more vectors.
  * ``route_partial_means`` — config 4 row-sharded (preferred): rank r computes
    the batch means of its ROW shard for every vector of the step (the
    retain-sampled FWHT restricted to those rows is 1/W of the Kerdock pass)
    and one all-to-all of means (K x rows per vector, ~1 GB per step instead
    of the retained columns) gives each vector owner complete means for the
    estimator's tail.
  * ``max_over_ranks``     — step time = max over ranks (device-timed).

Everything here is host logic; it is tested on CPU with the gloo backend
(tests/test_parallel_gloo.py) and runs on NCCL in bench.py.
"""
from __future__ import annotations

from typing import List, Tuple

import numpy as np


def vector_shard(rank: int, world: int, per_rank: int) -> Tuple[int, int]:
    """Weak scaling: rank r streams global vectors [r * per_rank, (r + 1) * per_rank)."""
    if not (0 <= rank < world) or per_rank < 0:
        raise ValueError("vector_shard: bad rank/world/per_rank")
    return rank * per_rank, per_rank


def strong_shard(rank: int, world: int, total: int) -> Tuple[int, int]:
    """Strong scaling split of `total` vectors (contiguous, sizes differ by at most 1)."""
    if not (0 <= rank < world) or total < 0:
        raise ValueError("strong_shard: bad rank/world/total")
    base, extra = divmod(total, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def basis_shards(nk: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous Kerdock-basis ranges per rank covering [0, nk) (sizes differ by at most 1)."""
    if nk < 0 or world < 1:
        raise ValueError("basis_shards: bad nk/world")
    return [strong_shard(r, world, nk) for r in range(world)]


def shard_element_range(basis_range: Tuple[int, int], d: int, ldc: int) -> Tuple[int, int]:
    """Element offsets [lo, hi) of a basis range inside the column-major sketch."""
    first, count = basis_range
    return first * d * ldc, (first + count) * d * ldc


class _CudaView:
    """Zero-copy device buffer exposed through __cuda_array_interface__ (for NCCL)."""

    def __init__(self, ptr: int, nelem: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (nelem,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def sketch_tensor(sk, torch_mod=None):
    """A flat torch view of the sketch's device columns (no copy)."""
    import torch
    nelem = sk.L * sk.column_stride
    typestr = "<f8" if sk.dtype == np.float64 else "<f4"
    return torch.as_tensor(_CudaView(sk.device_columns_ptr(), nelem, typestr), device=f"cuda:{sk.device}")


def allgather_basis_shards(full, world: int, rank: int, nk: int, d: int, ldc: int, group=None) -> None:
    """In-place all-gather of the Kerdock block of a flat sketch tensor `full`; each rank's own
    shard (parallel.basis_shards(nk, world)[rank]) must already be filled.

    Equal shards (nk % world == 0, e.g. 2048 bases over 1/2/4/8 GPUs) use one
    all_gather_into_tensor; otherwise (world = 3, 5, 6, 7 ...) every rank broadcasts its own
    contiguous byte range in turn, in place (no padding copy of a 137 GB sketch)."""
    import torch.distributed as dist
    if world == 1:
        return
    if nk % world == 0:
        per = (nk // world) * d * ldc
        kerdock = full[: nk * d * ldc]
        mine = kerdock[rank * per:(rank + 1) * per]
        dist.all_gather_into_tensor(kerdock, mine, group=group)
        return
    for src, rng in enumerate(basis_shards(nk, world)):
        lo, hi = shard_element_range(rng, d, ldc)
        if hi > lo:
            dist.broadcast(full[lo:hi], src=src if group is None else dist.get_global_rank(group, src), group=group)


def column_owner(ells: np.ndarray, shards: List[Tuple[int, int]], d: int, nk: int) -> np.ndarray:
    """Rank that computes column ell: the owner of its Kerdock basis, the last rank for the identity block."""
    ells = np.asarray(ells, dtype=np.int64)
    starts = np.array([first for first, _ in shards], dtype=np.int64)
    basis = ells // d
    owner = np.searchsorted(starts, basis, side="right") - 1
    # empty shards share a start with their successor: searchsorted picks the last of them, which is non-empty
    owner = np.where(basis >= nk, len(shards) - 1, owner)
    return owner.astype(np.int64)


class RoutingPlan:
    """Who computes and who receives every (vector, sample) column of a chunk.

    idx_all (B, N): the draws of every vector of the chunk (identical on every
    rank, fstg_draw_samples); vec_ranges[q] = (first, count) rows owned by rank
    q (contiguous, increasing). Columns travel grouped by destination rank and,
    within a destination, in (vector, sample) order."""

    def __init__(self, idx_all: np.ndarray, vec_ranges: List[Tuple[int, int]], shards: List[Tuple[int, int]], d: int,
                 nk: int, rank: int):
        idx_all = np.asarray(idx_all, dtype=np.int64)
        B, N = idx_all.shape
        world = len(vec_ranges)
        if len(shards) != world or not (0 <= rank < world):
            raise ValueError("RoutingPlan: ranks / shards mismatch")
        if sum(c for _, c in vec_ranges) != B or any(vec_ranges[q][0] != sum(c for _, c in vec_ranges[:q])
                                                     for q in range(world)):
            raise ValueError("RoutingPlan: vector ranges must tile [0, B) in rank order")
        src = column_owner(idx_all.ravel(), shards, d, nk)
        flat = idx_all.ravel()
        # send side: my columns in flat (vector, sample) order == grouped by destination
        mine = np.nonzero(src == rank)[0]
        self.send_ells = flat[mine]
        row_dst = np.repeat(np.arange(world), [c * N for _, c in vec_ranges])
        self.send_counts = np.bincount(row_dst[mine], minlength=world).astype(np.int64)
        # receive side: rows of my vectors, grouped by source rank, flat order inside a source
        first, count = vec_ranges[rank]
        lo, hi = first * N, (first + count) * N
        src_mine = src[lo:hi]
        order = np.argsort(src_mine, kind="stable")
        self.recv_positions = order.astype(np.int64)          # local row (v_local * N + j) of each received column
        self.recv_counts = np.bincount(src_mine, minlength=world).astype(np.int64)
        self.local_rows = count * N


def route_retained_columns(plan: RoutingPlan, sample_fn, ldc: int, dtype, device, group=None):
    """Computes this rank's columns (sample_fn(ells) -> (len, ldc) tensor), exchanges them with one
    all_to_all_single, and returns the (local_rows, ldc) gathered buffer of this rank's vectors."""
    import torch
    import torch.distributed as dist
    send = sample_fn(plan.send_ells) if len(plan.send_ells) else torch.empty((0, ldc), dtype=dtype, device=device)
    recv = torch.empty((int(plan.recv_counts.sum()), ldc), dtype=dtype, device=device)
    dist.all_to_all_single(recv, send, output_split_sizes=plan.recv_counts.tolist(),
                           input_split_sizes=plan.send_counts.tolist(), group=group)
    del send
    gathered = torch.empty((plan.local_rows, ldc), dtype=dtype, device=device)
    gathered.index_copy_(0, torch.from_numpy(plan.recv_positions).to(device), recv)
    return gathered


def route_partial_means(part, vec_ranges: List[Tuple[int, int]], row_ranges: List[Tuple[int, int]], rank: int,
                        ld: int, group=None):
    """part: (B_all, K, rows of my row shard) batch means of every vector for this rank's rows;
    vec_ranges[q] = (first, count) vectors owned by rank q, row_ranges[r] = (begin, end) rows of
    rank r's shard. Returns (B_mine, K + 1, ld) complete means of this rank's vectors (slot K
    left for mu), via one all_to_all_single: rank r sends rows-shard r of q's vectors to q."""
    import torch
    import torch.distributed as dist
    world = len(vec_ranges)
    B_all, K, h_me = part.shape
    first, count = vec_ranges[rank]
    # send: for every destination q its vectors' block of my rows (contiguous in part)
    send = part.contiguous()
    send_counts = [c * K * h_me for _, c in vec_ranges]
    recv_counts = [count * K * (row_ranges[r][1] - row_ranges[r][0]) for r in range(world)]
    recv = torch.empty(sum(recv_counts), dtype=part.dtype, device=part.device)
    dist.all_to_all_single(recv, send.view(-1), output_split_sizes=recv_counts, input_split_sizes=send_counts,
                           group=group)
    full = torch.zeros((count, K + 1, ld), dtype=part.dtype, device=part.device)
    off = 0
    for r in range(world):
        r0, r1 = row_ranges[r]
        n = recv_counts[r]
        full[:, :K, r0:r1] = recv[off:off + n].view(count, K, r1 - r0)
        off += n
    return full


def broadcast_matrix(a, src: int = 0, group=None):
    import torch.distributed as dist
    dist.broadcast(a, src=src, group=group)
    return a


def max_over_ranks(value: float, device=None, group=None) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
