"""Where a slow bench step spends its time: CUDA events around the select's
phases plus host timestamps, for 8 back-to-back C2 steps."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2501_07642_b200 as frr  # noqa: E402
from paper_2501_07642_b200 import _select as S  # noqa: E402
from paper_2501_07642_b200 import generation as G  # noqa: E402

M = 10**8
X = np.random.default_rng(2).standard_normal((1000, 64))
design = frr.DesignSpec(1000, 500, accept_prob=1e-3, max_draws=M, batch_size=10_000, root_seed=42)
kern = frr.precompute_precision(X, "exact")._kernel
stats = torch.empty(M, dtype=torch.float64, device="cuda")
ops, comm = S.DeviceSelectOps(), S.LocalComm()
log = []
orig_ub, orig_full = S._upper_bound_bits, S._select_full


def ub(*a, **k):
    log.append(("ub0", time.perf_counter()))
    r = orig_ub(*a, **k)
    log.append(("ub1", time.perf_counter()))
    return r


def full(*a, **k):
    log.append(("full0", time.perf_counter()))
    r = orig_full(*a, **k)
    log.append(("full1", time.perf_counter()))
    return r


S._upper_bound_bits, S._select_full = ub, full
for it in range(8):
    log.clear()
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    G.mc_stats_device(kern, design, 0, M, out=stats)
    h1 = time.perf_counter()
    S.select_k_smallest(stats, 0, 100_000, ops, comm)
    torch.cuda.synchronize()
    h2 = time.perf_counter()
    marks = " ".join(f"{n}={1e3 * (t - h0):.1f}" for n, t in log)
    print(f"step {it}: total {1e3 * (h2 - h0):.1f} ms, launch {1e3 * (h1 - h0):.2f}, {marks}", flush=True)
