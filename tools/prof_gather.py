"""Random 16 KiB column gathers: full 137.5 GB span vs small spans (TLB / page locality)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2105_05879_b200 import fst, parallel

a = np.random.default_rng(0).standard_normal((4096, 4096)).astype(np.float32)
sk = fst.preprocess(a)
t = parallel.sketch_tensor(sk).view(sk.L, sk.column_stride)
cnt = 200000  # 3.3 GB read per trial
out = torch.empty((cnt, sk.column_stride), device="cuda")
for span_cols in [sk.L, sk.L // 8, sk.L // 64, 65536, 8192]:
    idx = torch.randint(0, span_cols, (cnt,), device="cuda")
    sorted_idx, _ = torch.sort(idx)
    for name, ii in [("random", idx), ("sorted", sorted_idx)]:
        torch.index_select(t, 0, ii, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            torch.index_select(t, 0, ii, out=out)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        gb = cnt * sk.column_stride * 4 / 1e9
        print(f"span {span_cols * sk.column_stride * 4 / 1e9:9.2f} GB {name:6s}: read {gb / ms * 1e3:7.0f} GB/s "
              f"(read+write {2 * gb / ms * 1e3:7.0f} GB/s)")
