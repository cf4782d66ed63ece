"""One full C4 pool (2.33e9 ranks), for an ncu launch list."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2501_07642_b200 as frr  # noqa: E402

X = np.random.default_rng(4).standard_normal((34, 5))
pool = frr.enumerate_exact(X, frr.DesignSpec(34, 17, accept_prob=1e-3, mode="exact", enumeration_cap=3 * 10**9))
print(pool.n_accepted)
