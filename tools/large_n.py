"""MC pass-1 throughput across n (which tensor-core layout serves each shape)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_07642_b200 as frr
from paper_2501_07642_b200 import generation as G
for (n, d) in [(1000, 64), (2000, 64), (3000, 40), (5000, 64), (12000, 24), (2000, 1024), (3000, 333), (5000, 128)]:
    X = np.random.default_rng(1).standard_normal((n, d))
    design = frr.DesignSpec(n, n // 2, accept_prob=1e-3, max_draws=10**9, root_seed=5)
    kern = frr.precompute_precision(X, "exact")._kernel
    M = 1 << 20
    out = torch.empty(M, dtype=torch.float64, device="cuda")
    G.mc_stats_device(kern, design, 0, M, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); G.mc_stats_device(kern, design, 0, M, out); e1.record(); torch.cuda.synchronize()
    print(n, d, kern.tc_plan(), f"{M / e0.elapsed_time(e1) * 1e3:.3e} cand/s, draws/s {M * (n // 2) / e0.elapsed_time(e1) * 1e3:.3e}")
