"""Where randomization_test(find_fi=True) spends its time at C5 (n=5000,
1e6 keys): cProfile of one call after a warm-up call."""
import cProfile
import os
import pstats
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_07642_b200 as frr  # noqa: E402

m = 10**6
keys = np.column_stack([np.full(m, 5, dtype=np.uint64), 997 * np.arange(m, dtype=np.uint64)])
pool = frr.RandomizationPool(
    design=frr.DesignSpec(5000, 2500, accept_prob=1.0, max_draws=m * 997, batch_size=997, root_seed=5),
    stats=np.zeros(m), threshold_value=0.0, n_candidates=m * 997, accepted_indices=997 * np.arange(m), keys=keys)
X = np.random.default_rng(5).standard_normal((5000, 64))
obs = frr.batch_assignments(5, np.array([0], dtype=np.uint64), 5000, 2500)[0]
rng = np.random.default_rng(5)
y = X @ rng.standard_normal(64) + 1.0 * obs + 0.5 * rng.standard_normal(5000)
frr.randomization_test(obs, y, pool, find_fi=True)
for _ in range(3):
    t0 = time.perf_counter()
    frr.randomization_test(obs, y, pool, find_fi=True)
    print(f"wall {1e3 * (time.perf_counter() - t0):.2f} ms")
pr = cProfile.Profile()
pr.enable()
frr.randomization_test(obs, y, pool, find_fi=True)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
