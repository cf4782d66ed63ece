"""Where the public-API C2 call spends time beyond pass 1: cProfile of
monte_carlo_pool(X_host, design) at the bench config (top functions by
cumulative time), plus the wall time of three calls."""
import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_07642_b200 as frr  # noqa: E402

X = np.random.default_rng(2).standard_normal((1000, 64))
design = frr.DesignSpec(1000, 500, accept_prob=1e-3, max_draws=10**8, batch_size=10_000, root_seed=42)
frr.monte_carlo_pool(X, design)
torch.cuda.synchronize()
for _ in range(3):
    t0 = time.perf_counter()
    frr.monte_carlo_pool(X, design)
    print(f"wall {1e3 * (time.perf_counter() - t0):.2f} ms")
pr = cProfile.Profile()
pr.enable()
frr.monte_carlo_pool(X, design)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(28)
