"""Config-3 preprocessing time (n = m = 4096 fp32, 137.5 GB sketch) under FSTG_PRE_LOCKSTEP
settings (experiment switch: clusters of 2 / 4 row tiles with one relaxed cluster barrier per
basis before the write-back), alternated on one box. Tools only. The switch was measured and
removed (profiles/r01_preprocess_writepath.txt); against the current build all three settings
run the default kernel."""
import os
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2105_05879_b200 import fst  # noqa: E402

a = np.random.default_rng(0).standard_normal((4096, 4096)).astype(np.float32)
ref = None
for rep in range(2):
    for mode in ("0", "2", "4"):
        os.environ["FSTG_PRE_LOCKSTEP"] = mode
        sk = fst.preprocess(a)
        col = np.concatenate([sk.column(ell) for ell in (0, 12345, 4096 * 1000 + 17, 4096 * 2047 + 4095)])
        if ref is None:
            ref = col
        assert col.tobytes() == ref.tobytes(), mode
        print(f"lockstep={mode} preprocess_ms={sk.preprocess_ms:.2f} TB/s={sk.L * 4096 * 4 / sk.preprocess_ms / 1e9:.2f}",
              flush=True)
        sk.close()
