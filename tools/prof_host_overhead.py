"""Host-side cost of one fstg_transform_batch call at config-1 size (64 vectors, n = 256 fp64
STRICT, device-resident inputs/outputs), tools only: wall time of enqueueing 200 calls
without synchronising vs the device time of the same 200 calls (CUDA events)."""
import sys
import time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2105_05879_b200 import fst, generators  # noqa: E402

prob = generators.config1_problem(B=64, seed=1, device="cuda:0") if hasattr(generators, "config1_problem") else None
rng = np.random.default_rng(0)
if prob is None:
    a = torch.from_numpy(np.linalg.qr(rng.standard_normal((256, 256)))[0]).cuda()
    X = torch.from_numpy(rng.standard_normal((64, 256))).cuda()
else:
    a, X = prob.A, prob.X
sk = fst.preprocess(a)
p = fst.StreamParams(epsilon=0.1, s=8, J=375, K=2)
seeds = torch.arange(64, dtype=torch.int64, device="cuda")
want = fst.candidate_count(8, 10, 256)
out = fst.BatchResult(torch.zeros(64, dtype=torch.int32, device="cuda"), torch.zeros((64, want), dtype=torch.int32,
                      device="cuda"), torch.zeros((64, want), dtype=torch.float64, device="cuda"))
for prof in (False, True):
    fst.profile_enable(prof)
    for _ in range(20):
        fst.transform_batch(sk, X, p, seeds=seeds, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(200):
        fst.transform_batch(sk, X, p, seeds=seeds, out=out)
    t_host = time.perf_counter() - t0
    e1.record()
    torch.cuda.synchronize()
    t_all = time.perf_counter() - t0
    print(f"profile={prof}: host enqueue {t_host / 200 * 1e6:.1f} us/call, device {e0.elapsed_time(e1) / 200 * 1e3:.1f} "
          f"us/call, wall {t_all / 200 * 1e6:.1f} us/call, {64 * 200 / t_all:.0f} vectors/s")
