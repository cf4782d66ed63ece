"""One C4 public-API pool build (exact n=34, t=17, d=5, p=1e-3), for ncu captures."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_07642_b200 as frr  # noqa: E402

X = np.random.default_rng(4).standard_normal((34, 5))
pool = frr.enumerate_exact(X, frr.DesignSpec(34, 17, accept_prob=1e-3, mode="exact", enumeration_cap=3 * 10**9))
print(pool.n_accepted, pool.threshold_value)
