"""Host-side profile of the warm C1 public-API job (pool + test + FI)."""
import cProfile
import os
import pstats
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2501_07642_b200 as frr  # noqa: E402

rng = np.random.default_rng(1)
X = rng.standard_normal((20, 5))
design = frr.DesignSpec(20, 10, accept_prob=0.01, mode="exact", batch_size=10_000)
beta, noise = rng.standard_normal(5), 0.5 * rng.standard_normal(20)


def job():
    pool = frr.enumerate_exact(X, design)
    obs = pool.assignments[0]
    y = X @ beta + 1.0 * obs + noise
    return frr.randomization_test(obs, y, pool, find_fi=True)


job()
for _ in range(2):
    t0 = time.perf_counter()
    job()
    print("warm wall ms", (time.perf_counter() - t0) * 1e3)
pr = cProfile.Profile()
pr.enable()
job()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
