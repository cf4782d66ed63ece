"""Host-side profile of the full C4 pool (2.33e9 ranks): warm second call."""
import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2501_07642_b200 as frr  # noqa: E402

X = np.random.default_rng(4).standard_normal((34, 5))
design = frr.DesignSpec(34, 17, accept_prob=1e-3, mode="exact", enumeration_cap=3 * 10**9)
for _ in range(2):
    t0 = time.perf_counter()
    pool = frr.enumerate_exact(X, design)
    torch.cuda.synchronize()
    print("wall s", time.perf_counter() - t0, pool.n_accepted)
pr = cProfile.Profile()
pr.enable()
pool = frr.enumerate_exact(X, design)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
