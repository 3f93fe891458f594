"""Retain-sampled preprocessing (design-only sketches, fstg_sample_columns) and
the gathered-column transform (stream.hpp:184-191, 235-236) — the path that
makes config 4 (n = 16384, 8.8 TB sketch) computable. GPU."""
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


def _idx(L, count, seed, extra=()):
    rng = np.random.default_rng(seed)
    idx = rng.integers(0, L, size=count)
    return np.concatenate([idx, np.array(extra, dtype=np.int64), idx[:5]]).astype(np.int64)  # + duplicates


@pytest.mark.parametrize("m,n,dtype", [(40, 256, np.float64), (33, 1000, np.float32), (7, 4096, np.float32),
                                       (256, 256, np.float64), (5, 60, np.float32)])
def test_sample_columns_equal_sketch_columns(fst, m, n, dtype):
    a = np.random.default_rng(m + n).standard_normal((m, n)).astype(dtype)
    sk = fst.preprocess(a)
    idx = _idx(sk.L, 300, 1, extra=[0, sk.L - 1, sk.L - sk.d, sk.L - sk.d + n - 1])
    got = fst.sample_columns(sk, idx)
    for j, ell in enumerate(idx):
        assert got[j, :m].tobytes() == sk.column(int(ell)).tobytes(), (j, ell)
    des = fst.preprocess_design(a)
    got2 = fst.sample_columns(des, idx)
    assert got2[:, :m].tobytes() == got[:, :m].tobytes()
    with pytest.raises(ValueError):
        des.column(0)
    with pytest.raises(ValueError):
        fst.transform_batch(des, np.zeros((1, n), dtype=dtype), fst.StreamParams(epsilon=0.1, s=1, J=2, K=2))
    with pytest.raises(IndexError):
        fst.sample_columns(des, np.array([sk.L], dtype=np.int64))


def test_gathered_transform_matches_sketch_and_oracle(fst, orc):
    import torch
    a = orc.gen_orthogonal(256, 31)
    sk, des, ref = fst.preprocess(a), fst.preprocess_design(a), orc.preprocess(a)
    B, J, K = 8, 60, 3
    X = np.stack([orc.gen_exact_sparse(a, 8, orc.gen_seed(v))[0] for v in range(B)])
    seeds = np.array([orc.stream_seed(v) for v in range(B)], dtype=np.uint64)
    p = fst.StreamParams(epsilon=0.1, s=8, J=J, K=K)
    idx = fst.draw_samples(sk, p, seeds=seeds)                        # (B, N)
    cols = torch.from_numpy(fst.sample_columns(des, idx.ravel())).cuda()
    g = fst.transform_gathered_batch(des, X, p, idx, cols, candidates=True, mu=True)
    d = fst.transform_batch(sk, X, p, seeds=seeds, candidates=True, mu=True)
    for v in range(B):
        rg, rd = g.result(v), d.result(v)
        r = orc.transform(ref, X[v], orc.StreamParams(epsilon=0.1, s=8, J=J, K=K, seed=int(seeds[v])))
        for res in (rg, rd):
            assert np.array_equal(res.mu, r.mu)
            assert res.candidate_set.tolist() == r.candidate_set.tolist()
            assert res.support.tolist() == r.support.tolist()
            np.testing.assert_allclose(res.values, r.values, rtol=1e-12)


@pytest.mark.parametrize("m,n", [(2048, 4096), (600, 4000), (64, 16384)])
def test_sample_columns_many_rows_sparse_bases(fst, orc, m, n):
    """Many row tiles -> many bases per CTA (bpc up to 256) with most bases
    holding no request: the visited-basis walk and its sign-word prefetch."""
    import torch
    a = torch.randn(m, n, dtype=torch.float64, device="cuda:0", generator=torch.Generator("cuda:0").manual_seed(m))
    a32 = a.float().contiguous()
    des = fst.preprocess_design(a32)
    idx = _idx(des.L, 40, m, extra=[0, 1, des.d, des.L - des.d - 1, des.L - des.d, des.L - 1])
    got = fst.sample_columns(des, idx)[:, :m].astype(np.float64)
    S = torch.from_numpy(orc.design_columns(des.k, n, idx)).cuda()
    expect = (S @ a32.double().T).cpu().numpy()
    err = np.abs(got - expect).max(axis=1)
    scale = np.abs(expect).max(axis=1)
    assert np.all(err <= 2e-5 * np.maximum(scale, 1.0)), (err.max(), np.argmax(err))


def test_config4_shape_spot_check(fst, orc):
    """n = 16384 (k = 14, the 8.8 TB design): sampled columns of a design-only
    sketch vs A s_ell in fp64, and three vectors through the gathered transform
    vs the oracle's draw_and_gather path on the same columns."""
    import torch
    from paper_2105_05879_b200 import generators
    n = 16384
    A64 = generators.iid_gaussian(n, 1024, "cuda:0")
    A32 = A64.float().contiguous()
    des = fst.preprocess_design(A32)
    assert des.L == 134234112 and des.k == 14
    idx = _idx(des.L, 64, 7, extra=[des.L - 1, des.L - des.d])
    got = fst.sample_columns(des, idx)
    S = torch.from_numpy(orc.design_columns(14, n, idx)).cuda()     # (count, n) design vectors s_ell
    expect = (S @ A32.double().T).cpu().numpy()                       # column ell = A s_ell
    err = np.abs(got.astype(np.float64) - expect).max(axis=1)
    scale = np.abs(expect).max(axis=1) + 1e-30
    assert np.all(err <= 2e-5 * np.maximum(scale, 1.0)), err.max()
    # three vectors, J = 100, K = 2, s = 64, eps = 0.05 (config 4 parameters, shorter N)
    prob = generators.config2_problem  # noqa: F841 (config 4 uses the same A^-1 y generator at n = 16384)
    B = 3
    g_seeds, st_seeds = generators.trial_seeds(11, 0, B)
    Y = generators.sparse_targets(g_seeds, n, 64, value_kind=1)
    lu = torch.linalg.lu_factor(A64)
    X64 = torch.linalg.lu_solve(*lu, torch.from_numpy(Y).cuda().T).T
    X64 = X64 / torch.linalg.vector_norm(X64, dim=1, keepdim=True)
    X = X64.float().contiguous()
    p = fst.StreamParams(epsilon=0.05, s=64, J=100, K=2)
    ind = fst.draw_samples(des, p, seeds=st_seeds)
    cols = torch.from_numpy(fst.sample_columns(des, ind.ravel())).cuda()
    out = fst.transform_gathered_batch(des, X, p, ind, cols, candidates=True, mu=True)
    a_host = A32.double().cpu().numpy()
    for v in range(B):
        gathered = cols[v * 200:(v + 1) * 200, :n].double().cpu().numpy()
        x = X[v].double().cpu().numpy()
        r = orc.transform_gathered(a_host, x, orc.StreamParams(epsilon=0.05, s=64, J=100, K=2), ind[v], gathered)
        g = out.result(v)
        np.testing.assert_allclose(g.mu, r.mu, rtol=1e-4, atol=1e-5)
        assert g.support.tolist() == r.support.tolist()
        np.testing.assert_allclose(g.values, r.values, rtol=1e-5)


def test_route_retained_columns_nccl_single_rank(fst, orc):
    """The config-4 multi-GPU routing (RoutingPlan + NCCL all_to_all_single +
    scatter) on a one-rank NCCL group with the real fstg_sample_columns: the
    routed buffer equals the direct draw_and_gather columns."""
    import os
    import socket
    import torch
    import torch.distributed as dist
    from paper_2105_05879_b200 import parallel
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda:0"))
    try:
        a = torch.randn(300, 1000, device="cuda:0", dtype=torch.float32)
        des = fst.preprocess_design(a)
        idx_all = np.random.default_rng(2).integers(0, des.L, size=(6, 50))
        nk = des.d // 2
        plan = parallel.RoutingPlan(idx_all, [(0, 6)], parallel.basis_shards(nk, 1), des.d, nk, 0)

        def sample_fn(ells):
            buf = torch.empty((len(ells), des.column_stride), dtype=torch.float32, device="cuda:0")
            fst.sample_columns(des, ells, out=buf)
            return buf

        got = parallel.route_retained_columns(plan, sample_fn, des.column_stride, torch.float32, "cuda:0")
        want = fst.sample_columns(des, idx_all.ravel())
        assert np.array_equal(got.cpu().numpy(), want)
    finally:
        dist.destroy_process_group()


def _same(a, b):
    import torch
    a = a.cpu().numpy() if isinstance(a, torch.Tensor) else a
    b = b.cpu().numpy() if isinstance(b, torch.Tensor) else b
    return a.shape == b.shape and a.tobytes() == b.tobytes()


@pytest.mark.parametrize("m,n,dtype,mode,row_block", [(200, 256, np.float32, 0, 64), (200, 256, np.float32, 0, 0),
                                                      (130, 256, np.float64, 0, 40), (300, 1000, np.float32, 1, 96),
                                                      (64, 4096, np.float32, 0, 16)])
def test_transform_design_batch_equals_full_sketch(fst, m, n, dtype, mode, row_block):
    """Row-blocked design-only transform (per row block: retain-sampled FWHT of those
    rows + PARTIAL stream; then TAIL): every output bit-identical to the full-sketch
    transform, because each row's batch sum runs over j in the same order."""
    import torch
    rng = np.random.default_rng(m + n)
    a = rng.standard_normal((m, n)).astype(dtype)
    sk, des = fst.preprocess(a), fst.preprocess_design(a)
    B = 37
    X = torch.from_numpy(rng.standard_normal((B, n)).astype(dtype)).cuda()
    seeds = torch.from_numpy(rng.integers(0, 2**63, size=B, dtype=np.int64)).cuda()
    p = fst.StreamParams(epsilon=0.5, s=3, J=23, K=3, mode=mode)
    ref = fst.transform_batch(sk, X, p, seeds=seeds, candidates=True, mu=True)
    got = fst.transform_design_batch(des, X, p, seeds=seeds, row_block=row_block, candidates=True, mu=True)
    for f in ("counts", "support", "values", "candidates", "mu"):
        assert _same(getattr(ref, f), getattr(got, f)), f
    with pytest.raises(ValueError):
        fst.transform_design_batch(des, X.cpu(), p, seeds=seeds)
    sk.close()


def test_transform_design_batch_config4_shape(fst):
    """n = 16384 (k = 14): the row-blocked path equals the gathered-column path
    (fstg_sample_columns of whole columns + fstg_transform_gathered_batch) bit for bit."""
    import torch
    from paper_2105_05879_b200 import generators
    n, m = 16384, 256
    A = generators.iid_gaussian(n, 1024, "cuda:0")[:m].float().contiguous()
    des = fst.preprocess_design(A)
    B = 3
    X = torch.randn(B, n, device="cuda:0", generator=torch.Generator("cuda:0").manual_seed(1))
    X = (X / torch.linalg.vector_norm(X, dim=1, keepdim=True)).contiguous()
    seeds = torch.tensor([11, 12, 13], dtype=torch.int64, device="cuda:0")
    p = fst.StreamParams(epsilon=0.01, s=8, J=40, K=2)
    ind = fst.draw_samples(des, p, seeds=seeds.cpu().numpy().view(np.uint64))
    cols = torch.from_numpy(fst.sample_columns(des, ind.ravel())).cuda()
    ref = fst.transform_gathered_batch(des, X, p, ind, cols, candidates=True, mu=True)
    got = fst.transform_design_batch(des, X, p, seeds=seeds, row_block=96, candidates=True, mu=True)
    for f in ("counts", "support", "values", "candidates", "mu"):
        assert _same(getattr(ref, f), getattr(got, f)), f


@pytest.mark.parametrize("dtype,mode", [(np.float32, 0), (np.float64, 0)])
def test_row_sharded_partial_means_equal_design_batch(fst, dtype, mode):
    """Two 'ranks' emulated in one process: each computes the batch means of its row
    shard for every vector (fstg_design_partial_means), the shards are assembled per
    vector owner (what parallel.route_partial_means does over NCCL), and
    fstg_transform_from_means gives outputs bit-identical to fstg_transform_design_batch."""
    import torch
    rng = np.random.default_rng(8)
    m, n, B = 200, 256, 6
    a = rng.standard_normal((m, n)).astype(dtype)
    des = fst.preprocess_design(a)
    X = torch.from_numpy(rng.standard_normal((B, n)).astype(dtype)).cuda()
    seeds = torch.from_numpy(rng.integers(0, 2**63, size=B, dtype=np.int64)).cuda()
    p = fst.StreamParams(epsilon=0.5, s=3, J=17, K=3, mode=mode)
    ref = fst.transform_design_batch(des, X, p, seeds=seeds, candidates=True, mu=True)
    rows = [(0, 96), (96, 200)]
    vecs = [(0, 4), (4, 2)]
    parts = [fst.design_partial_means(des, X, p, seeds=seeds, row_begin=r0, row_end=r1, row_block=40)
             for r0, r1 in rows]
    ld = (m + 3) // 4 * 4
    for first, count in vecs:
        full = torch.zeros((count, p.K + 1, ld), dtype=X.dtype, device="cuda:0")
        for (r0, r1), part in zip(rows, parts):
            full[:, :p.K, r0:r1] = part[first:first + count]
        got = fst.transform_from_means(des, X[first:first + count], p, full, candidates=True, mu=True)
        for f in ("counts", "support", "values", "candidates", "mu"):
            assert _same(getattr(ref, f)[first:first + count], getattr(got, f)), f


def test_design_transform_returns_pool_memory(fst):
    """After a design-only transform whose transient column buffers fill most of HBM
    (auto row blocks: ~70% of free memory) the library's pool is trimmed, so the
    caller can allocate most of HBM again."""
    import torch
    rng = np.random.default_rng(4)
    a = rng.standard_normal((4096, 1024)).astype(np.float32)
    des = fst.preprocess_design(a)
    B = 16384
    X = torch.from_numpy(rng.standard_normal((B, 1024)).astype(np.float32)).cuda()
    p = fst.StreamParams(epsilon=0.5, s=4, J=375, K=2)
    out = fst.transform_design_batch(des, X, p, seeds=np.arange(B, dtype=np.uint64))
    torch.cuda.synchronize()
    assert int(out.counts.max()) >= 0
    free, total = torch.cuda.mem_get_info()
    assert free > 0.5 * total, (free, total)
    # retained pool: the scratch stays cached (and is reused) until retain is cleared
    fst.set_pool_retain(True)
    try:
        for _ in range(2):
            fst.transform_design_batch(des, X, p, seeds=np.arange(B, dtype=np.uint64))
        torch.cuda.synchronize()
        free_kept, _ = torch.cuda.mem_get_info()
        assert free_kept < 0.5 * total, (free_kept, total)
    finally:
        fst.set_pool_retain(False)
    free, _ = torch.cuda.mem_get_info()
    assert free > 0.5 * total, (free, total)


def _with_cluster(cl, fn):
    """Runs fn() with the k = 14 cluster-merged retain write-back at cluster size cl
    (4 or 8 CTAs) or disabled (0) (FSTG_RETAIN_CLUSTER, read by the launcher at every call)."""
    import os
    old = os.environ.get("FSTG_RETAIN_CLUSTER")
    os.environ["FSTG_RETAIN_CLUSTER"] = str(cl)
    try:
        return fn()
    finally:
        if old is None:
            del os.environ["FSTG_RETAIN_CLUSTER"]
        else:
            os.environ["FSTG_RETAIN_CLUSTER"] = old


@pytest.mark.parametrize("m,cl,ws", [(77, 8, 1), (8, 8, 1), (3, 8, 1), (77, 4, 1), (6, 4, 1), (77, 4, 0), (9, 8, 0)])
def test_retain_cluster_merge_bit_identical(fst, orc, m, cl, ws, monkeypatch):
    """k = 14 (n = 5000 pads to d = 16384): the 8-CTA cluster write-back (rows
    merged into 32-byte column segments through distributed shared memory) gives
    the same bits as the per-row write-back, with ragged row counts (m not a
    multiple of 8, fewer rows than a cluster), a basis holding more requests than
    the shared-memory record buffer (chunked), duplicates and identity columns;
    and both match A s_ell in fp64. ws selects the warp-specialised kernel
    (default) or the single-warpgroup merge (FSTG_RETAIN_WS=0)."""
    import torch
    monkeypatch.setenv("FSTG_RETAIN_WS", str(ws))
    n = 5000
    rng = np.random.default_rng(m)
    a32 = torch.from_numpy(rng.standard_normal((m, n)).astype(np.float32)).cuda()
    des = fst.preprocess_design(a32)
    assert des.k == 14
    d = des.d
    dense = 3 * d + rng.integers(0, d, size=2500)              # 2500 requests in one basis (> 1024 records)
    idx = np.concatenate([_idx(des.L, 3000, 5, extra=[0, d - 1, des.L - d, des.L - 1]), dense]).astype(np.int64)
    on = _with_cluster(cl, lambda: fst.sample_columns(des, idx))
    off = _with_cluster(0, lambda: fst.sample_columns(des, idx))
    assert on[:, :m].tobytes() == off[:, :m].tobytes()
    S = torch.from_numpy(orc.design_columns(14, n, idx[::37])).cuda()
    expect = (S @ a32.double().T).cpu().numpy()
    err = np.abs(on[::37, :m].astype(np.float64) - expect).max(axis=1)
    assert np.all(err <= 2e-5 * np.maximum(np.abs(expect).max(axis=1), 1.0)), err.max()


def test_retain_cluster_partial_means_row_offsets(fst):
    """Row-sharded partial means at k = 14 with row ranges that are not multiples
    of the cluster size: cluster and per-row write-back are bit-identical."""
    import torch
    rng = np.random.default_rng(21)
    m, n, B = 150, 4500, 3
    a = torch.from_numpy(rng.standard_normal((m, n)).astype(np.float32)).cuda()
    des = fst.preprocess_design(a)
    X = torch.from_numpy(rng.standard_normal((B, n)).astype(np.float32)).cuda()
    seeds = torch.from_numpy(rng.integers(0, 2**63, size=B, dtype=np.int64)).cuda()
    p = fst.StreamParams(epsilon=0.5, s=3, J=40, K=2)
    run = lambda: fst.design_partial_means(des, X, p, seeds=seeds, row_begin=13, row_end=141, row_block=40)  # noqa: E731
    off = _with_cluster(0, run)
    for cl in (4, 8):
        assert torch.equal(_with_cluster(cl, run), off), cl


def test_config4_retained_columns_bit_exact(fst, orc):
    """n = 16384 (k = 14, the 8.8 TB design): every retained value of the warp-specialised,
    cluster-merged retain kernel is bit-identical to the float restatement of the reference's
    per-basis block (oracle.kerdock_block, sketch.hpp:171-196) — not just within 2e-5 of A s_ell."""
    n, m, d = 16384, 40, 16384
    rng = np.random.default_rng(14)
    a32 = (rng.standard_normal((m, n)) / np.sqrt(n)).astype(np.float32)
    des = fst.preprocess_design(a32)
    bases = [0, 1, 77, 4095, 4096, 8191]
    ells = [int(s) * d + int(w) for s in bases for w in rng.integers(0, d, size=4)]
    ells += [des.L - 1, des.L - d + 5]                          # identity block
    got = fst.sample_columns(des, np.array(ells, dtype=np.int64))[:, :m]
    blocks = {s: orc.kerdock_block(a32, s, np.float32) for s in bases}
    for j, ell in enumerate(ells):
        if ell < des.kerdock_bases() * d:
            ref = blocks[ell // d][ell % d]
        else:
            w = ell - des.kerdock_bases() * d
            ref = (np.float32(128.0) * a32[:, w]) if w < n else np.zeros(m, np.float32)
        assert got[j].tobytes() == ref.tobytes(), ell


def test_config4_design_transform_bit_exact_vs_kernel_order(fst, orc):
    """The config-4 transform (row-blocked design path: retain-sampled FWHT rows + PARTIAL batch
    means, then TAIL) at n = 16384 bit-exact, vector by vector, against the FAST kernels'
    restated arithmetic on the retained columns."""
    import torch
    n, m, B = 16384, 48, 160
    rng = np.random.default_rng(41)
    a32 = (rng.standard_normal((m, n)) / np.sqrt(n)).astype(np.float32)
    des = fst.preprocess_design(a32)
    X = rng.standard_normal((B, n))
    X = (X / np.linalg.norm(X, axis=1, keepdims=True)).astype(np.float32)
    seeds = np.array([orc.stream_seed(13000 + v) for v in range(B)], dtype=np.uint64)
    p = fst.StreamParams(epsilon=0.02, s=2, J=60, K=2)
    Xd = torch.from_numpy(X).cuda()
    out = fst.transform_design_batch(des, Xd, p, seeds=seeds, row_block=16, candidates=True, mu=True)
    idx = fst.draw_samples(des, p, seeds=seeds)
    mu, cand = out.mu.cpu().numpy(), out.candidates.cpu().numpy()
    counts, sup, vals = out.counts.cpu().numpy(), out.support.cpu().numpy(), out.values.cpu().numpy()
    for v in (0, 1, 79, 147, 148, 159):
        cols = fst.sample_columns(des, idx[v])[:, :m]
        r = orc.transform_gathered_fast_order(a32, X[v], orc.StreamParams(epsilon=0.02, s=2, J=60, K=2), idx[v],
                                              cols)
        assert mu[v].tobytes() == r.mu.tobytes(), v
        assert cand[v].tolist() == r.candidate_set.tolist(), v
        assert sup[v, :counts[v]].tolist() == r.support.tolist(), v
        assert vals[v, :counts[v]].tobytes() == r.values.tobytes(), v
