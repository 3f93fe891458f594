import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2105_05879_b200 import fst
rng = np.random.default_rng(3)
t0 = time.time()
a = torch.from_numpy(rng.standard_normal((4096, 4096)).astype(np.float32)).cuda()
ms = []
for i in range(40):
    sk = fst.preprocess(a)
    ms.append(sk.preprocess_ms)
    sk.close()
print("m=4096 x40: min %.2f median %.2f max %.2f ms" % (min(ms), sorted(ms)[20], max(ms)), flush=True)
for m in (8, 9, 100, 1000, 2047):
    b = torch.from_numpy(rng.standard_normal((m, 4000)).astype(np.float32)).cuda()
    for i in range(25):
        sk = fst.preprocess(b)
        sk.close()
    print("m=%d x25 ok" % m, flush=True)
# config-4 retain kernel, repeated
n = 16384
A = torch.randn(256, n, device="cuda") / 128
sk = fst.preprocess_design(A)
idx = torch.from_numpy(rng.integers(0, sk.L, size=8192 * 750, dtype=np.int64)).cuda()
out = torch.empty((idx.numel(), sk.column_stride), device="cuda", dtype=torch.float32)
ref = None
for i in range(12):
    fst.sample_columns(sk, idx, out=out)
    torch.cuda.synchronize()
    h = out[::997].clone()
    if ref is None:
        ref = h
    assert torch.equal(ref, h), i
print("k=14 retain x12 identical", flush=True)
print("total %.1f s" % (time.time() - t0))
