import time, numpy as np, torch, sys, os
sys.path.insert(0, os.getcwd())
import paper_2501_07642_b200 as frr
from paper_2501_07642_b200 import generation as G, balance as B
X = np.random.default_rng(2).standard_normal((1000, 64))
design = frr.DesignSpec(1000, 500, accept_prob=1e-3, max_draws=10**8, batch_size=10_000, root_seed=42)
frr.monte_carlo_pool(X, design); torch.cuda.synchronize()
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
t0 = time.perf_counter(); pool = frr.monte_carlo_pool(X, design); torch.cuda.synchronize(); t1 = time.perf_counter()
pr.disable()
print("e2e s", t1 - t0)
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
