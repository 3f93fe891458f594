"""Driver for ncu captures of the stream kernel at config 5 (n = 4096, s given, eps 0.2):
python tools/prof_c5.py [s] [B]. The second launch is the one to capture."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2105_05879_b200 import fst, generators  # noqa: E402

s = int(sys.argv[1]) if len(sys.argv) > 1 else 256
B = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
prob = generators.config5_problem(s, 0.2, B, seed=20251019, device="cuda:0")
sk = fst.preprocess(prob.A)
seeds = torch.from_numpy(prob.seeds.view(np.int64)).cuda()
p = fst.StreamParams(epsilon=0.2, s=s, J=375, K=2)
fst.profile_enable(True)
for _ in range(2):
    fst.profile_reset()
    out = fst.transform_batch(sk, prob.X, p, seeds=seeds)
    torch.cuda.synchronize()
    ms, n = fst.profile_read("stream")
    print(f"s={s} B={B}: stream {ms:.2f} ms, {B / ms * 1e3:.0f} vectors/s")
sk.close()
