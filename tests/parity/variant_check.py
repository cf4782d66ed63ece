"""Correctness + speed of one libfrr build (FRR_LIBRARY) on the C2 shape.
Usage: FRR_LIBRARY=... python tests/parity/variant_check.py [M]"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402

import paper_2501_07642_b200 as frr  # noqa: E402
from paper_2501_07642_b200 import generation as G  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 21
os.environ.setdefault("FRR_MC_PATH", "tensor_core")
X = np.random.default_rng(2).standard_normal((1000, 64))
design = frr.DesignSpec(1000, 500, accept_prob=1e-3, max_draws=M, batch_size=min(M, 10_000), root_seed=42)
kern = frr.precompute_precision(X, "exact")._kernel
st = G.mc_stats_device(kern, design, 0, 4096).cpu().numpy()
bal = O.balance_setup(X, O.precision(X, "exact"))
want = O.c_mc_stats(bal, 500, 42, 0, 4096)
bad = int((st.view(np.uint64) != want.view(np.uint64)).sum())
out = torch.empty(M, dtype=torch.float64, device="cuda")
G.mc_stats_device(kern, design, 0, M, out)
torch.cuda.synchronize()
times = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    G.mc_stats_device(kern, design, 0, M, out)
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
times.sort()
ms = times[2]  # median of 5
print(f"{os.path.basename(os.environ.get('FRR_LIBRARY', 'default'))}: mismatches={bad} rate={M / ms * 1e3:.3e} cand/s ({ms:.1f} ms)", flush=True)
