"""A/B helper: hash of sampled sketch columns (k = 12 fp32 paths) for bit-identity checks
between preprocessing kernel variants."""
import hashlib
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2105_05879_b200 import fst  # noqa: E402

for m, n in ((40, 4096), (64, 4000), (4096, 4096)):
    a = np.random.default_rng(m + n).standard_normal((m, n)).astype(np.float32)
    sk = fst.preprocess(a)
    rng = np.random.default_rng(1)
    idx = np.concatenate([np.arange(0, 3 * 4096), np.arange(sk.L - 2 * 4096, sk.L), rng.integers(0, sk.L, 60000)])
    cols = fst.sample_columns(sk, idx)
    print("m", m, "n", n, "ms", round(sk.preprocess_ms, 2), "sha", hashlib.sha256(cols.tobytes()).hexdigest()[:16],
          flush=True)
    sk.close()
