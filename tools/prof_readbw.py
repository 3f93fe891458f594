"""Read-bandwidth ceilings on the 137.5 GB sketch allocation: contiguous sum vs random-chunk sums."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2105_05879_b200 import fst, parallel

a = np.random.default_rng(0).standard_normal((4096, 4096)).astype(np.float32)
sk = fst.preprocess(a)
t = parallel.sketch_tensor(sk)


def timeit(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


view = t[: 8 * 2**30]  # 32 GiB contiguous
ms = timeit(lambda: view.sum())
print(f"contiguous read (sum 32 GiB): {view.numel() * 4 / ms / 1e6:7.0f} GB/s")
for chunk in [4096, 16384, 65536]:  # floats per chunk: 16 KiB, 64 KiB, 256 KiB
    nchunks = t.numel() // chunk
    cnt = (2**29) // chunk  # 2 GiB per trial
    idx = torch.randint(0, nchunks, (cnt,), device="cuda")
    v2 = t[: nchunks * chunk].view(nchunks, chunk)
    ms = timeit(lambda: v2.index_select(0, idx).sum())
    print(f"random {chunk * 4 // 1024:4d} KiB chunks gather+sum: {cnt * chunk * 4 / ms / 1e6:7.0f} GB/s read "
          f"(+ equal write of the gathered copy)")
