"""Small driver for ncu captures of the preprocessing kernels (same kernel code
path as n=4096, fewer rows so kernel replay does not have to save 137 GB)."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2105_05879_b200 import fst

m = int(sys.argv[1]) if len(sys.argv) > 1 else 256
a = np.random.default_rng(0).standard_normal((m, 4096)).astype(np.float32)
for _ in range(2):
    sk = fst.preprocess(a)
    print("preprocess_ms", sk.preprocess_ms, "GB", sk.L * m * 4 / 1e9, "GB/s", sk.L * m * 4 / sk.preprocess_ms / 1e6)
    sk.close()
