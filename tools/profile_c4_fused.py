"""The full C4 pool through the public API (n=34, t=17, d=5, p=1e-3): the
fused tiled pass 1 + narrowing (k_exact_tiled) and everything after it, for
ncu (-k regex:k_exact_tiled for the dominant kernel)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2501_07642_b200 as frr  # noqa: E402

X = np.random.default_rng(4).standard_normal((34, 5))
design = frr.DesignSpec(34, 17, accept_prob=1e-3, mode="exact", enumeration_cap=3 * 10**9)
pool = frr.enumerate_exact(X, design)
print(pool.n_accepted, pool.threshold_value)
