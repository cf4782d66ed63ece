"""Where the bench.py step's time goes: device time of pass 1, of the select,
and the host gaps between them (C2, 1e8 candidates)."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2501_07642_b200 as frr  # noqa: E402
from paper_2501_07642_b200 import generation as G  # noqa: E402
from paper_2501_07642_b200._select import DeviceSelectOps, LocalComm, select_k_smallest  # noqa: E402

M = 10**8
X = np.random.default_rng(2).standard_normal((1000, 64))
design = frr.DesignSpec(1000, 500, accept_prob=1e-3, max_draws=M, batch_size=10_000, root_seed=42)
kern = frr.precompute_precision(X, "exact")._kernel
stats = torch.empty(M, dtype=torch.float64, device="cuda")
ops, comm = DeviceSelectOps(), LocalComm()
for it in range(4):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    e[0].record()
    G.mc_stats_device(kern, design, 0, M, out=stats)
    e[1].record()
    h1 = time.perf_counter()
    res = select_k_smallest(stats, 0, 100_000, ops, comm)
    e[2].record()
    torch.cuda.synchronize()
    h2 = time.perf_counter()
    print(f"pass1 dev {e[0].elapsed_time(e[1]):.2f} ms, select dev {e[1].elapsed_time(e[2]):.2f} ms, "
          f"host launch {1e3 * (h1 - h0):.2f} ms, host total {1e3 * (h2 - h0):.2f} ms")
