"""Write-path experiment: full FWHT vs FWHT skipped (same store pattern) vs contiguous zero-fill."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2105_05879_b200 import fst, parallel

a = np.random.default_rng(0).standard_normal((4096, 4096)).astype(np.float32)
sk = fst.preprocess(a)
print("fwht default ms", sk.preprocess_ms, "GB/s", sk.L * 4096 * 4 / sk.preprocess_ms / 1e6)
t = parallel.sketch_tensor(sk)
for _ in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); t.zero_(); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print("contiguous zero-fill ms", ms, "GB/s", t.numel() * 4 / ms / 1e6)
sk.close()
os.environ["FSTG_FWHT_STORE"] = "nofwht"
sk = fst.preprocess(a)
print("nofwht (same pattern, no math) ms", sk.preprocess_ms, "GB/s", sk.L * 4096 * 4 / sk.preprocess_ms / 1e6)
