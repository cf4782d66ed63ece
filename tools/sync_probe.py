"""Which host-side call of the select blocks behind a running pass 1?  Each
probe runs right after a 100 ms pass-1 launch; a probe that returns after
~100 ms waited for the GPU."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_07642_b200 as frr  # noqa: E402
from paper_2501_07642_b200 import _select as S  # noqa: E402
from paper_2501_07642_b200 import generation as G  # noqa: E402
from paper_2501_07642_b200._select import DeviceSelectOps, LocalComm  # noqa: E402

X = np.random.default_rng(2).standard_normal((1000, 64))
design = frr.DesignSpec(1000, 500, accept_prob=1e-3, max_draws=10**8, batch_size=10_000, root_seed=42)
kern = frr.precompute_precision(X, "exact")._kernel
stats = torch.empty(10**8, dtype=torch.float64, device="cuda")
G.mc_stats_device(kern, design, 0, 10**8, out=stats)
torch.cuda.synchronize()
ops = DeviceSelectOps()
ring = torch.empty((8, 4), dtype=torch.int64, pin_memory=True)
small = torch.ones(4, dtype=torch.int64, device="cuda")
idx_map = torch.arange(1000, device="cuda")
idx = torch.randint(0, 1000, (100,), device="cuda")


def probe(name, fn):
    out = []
    for _ in range(3):
        G.mc_stats_device(kern, design, 0, 10**8, out=stats)
        t0 = time.perf_counter()
        fn()
        out.append(1e3 * (time.perf_counter() - t0))
        torch.cuda.synchronize()
    print(f"{name:28s} " + " ".join(f"{x:8.2f}" for x in out) + " ms", flush=True)


probe("nothing", lambda: None)
probe("d2h pinned ring slice", lambda: ring[1, :1].copy_(small[:1], non_blocking=True))
probe("d2h pinned fresh", lambda: torch.empty(1, dtype=torch.int64, pin_memory=True).copy_(small[:1], non_blocking=True))
probe("gather idx_map[idx]", lambda: idx_map[idx.clamp(0, 999)])
probe("masked_fill", lambda: small.masked_fill(small > small[:1], 0))
probe("ops.init", lambda: ops.init(5, stats.device))
st = ops.init(100, stats.device)
probe("ops.hist", lambda: ops.hist(stats[:1000], st, 0))
probe("strided sample", lambda: stats[::95][:1 << 20].contiguous())
probe("set_threshold_from", lambda: ops.set_threshold_from(ops.init(5, stats.device), st))
probe("select_start", lambda: S.select_start(stats, 0, 100_000, ops, LocalComm(), m_total=10**8))
