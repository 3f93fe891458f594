"""Driver for the k = 14 retain-sampled Kerdock pass (config 4's hot kernel), tools only.

python tools/prof_k14.py [rows] [requests]
  rows     rows of A (n = 16384 columns, so k = 14); default 1024
  requests sampled column indices (uniform over L, seeded); default 8192 * 750;
           0 = one request per Kerdock basis (FWHT cost alone)
Prints the FWHT kernel's device time (library CUDA-event scope) and the add rate
scaled to the full pass (all 8192 Kerdock bases x 16384 rows).
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2105_05879_b200 import fst  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
nreq = int(sys.argv[2]) if len(sys.argv) > 2 else 8192 * 750
n, k = 16384, 14
d = 1 << k
a = torch.randn(rows, n, device="cuda", dtype=torch.float32) / np.sqrt(n)
sk = fst.preprocess_design(a)
L = sk.L
if nreq == 0:  # one request per Kerdock basis: every basis visited, negligible copy work
    idx = torch.arange(0, (d // 2) * d, d, dtype=torch.int64, device="cuda")
    nreq = idx.numel()
else:
    idx = torch.from_numpy(np.random.default_rng(7).integers(0, L, size=nreq, dtype=np.int64)).cuda()
out = torch.empty((nreq, sk.column_stride), device="cuda", dtype=torch.float32)
fst.profile_enable(True)
for rep in range(3):
    fst.profile_reset()
    fst.sample_columns(sk, idx, out=out)
    torch.cuda.synchronize()
    ms, _ = fst.profile_read("sample_columns_fwht")
    adds = (d // 2) * rows * d * k
    full_ms = ms * 16384 / rows
    print(f"rows={rows} requests={nreq} fwht_ms={ms:.2f} -> full-pass-equivalent {full_ms:.0f} ms, "
          f"{adds / ms / 1e9:.2f} Tadd/s")
try:  # variant builds with -DFSTG_WS_PROF: per-phase cycles of one butterfly / copy thread per CTA
    import ctypes
    fn = fst.lib().fstg_debug_wsprof
    buf = (ctypes.c_ulonglong * 16)()
    fn(buf)  # discard the warm-up accumulations
    fst.sample_columns(sk, idx, out=out)
    torch.cuda.synchronize()
    fn(buf)
    nbr = (d // 2) * rows  # basis-rows of the launch
    print("wsprof cycles per basis-row: butterfly " + " ".join(f"{buf[i] / nbr:.0f}" for i in range(8))
          + " | copy " + " ".join(f"{buf[8 + i] / nbr:.0f}" for i in range(8)))
except AttributeError:
    pass
sk.close()
