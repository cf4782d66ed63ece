"""Correctness + speed of one libfrr build (FRR_LIBRARY) on the C3 shape."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402

import paper_2501_07642_b200 as frr  # noqa: E402
from paper_2501_07642_b200 import generation as G  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
X = np.random.default_rng(3).standard_normal((2000, 1024))
design = frr.DesignSpec(2000, 1000, accept_prob=1e-4, max_draws=M, batch_size=min(M, 10_000), root_seed=43,
                        precision_mode="ridge")
kern = frr.precompute_precision(X, "ridge")._kernel
st = G.mc_stats_device(kern, design, 0, 512).cpu().numpy()
want = O.c_mc_stats(O.Balance(kern._zq, kern._inv_scale_sq), 1000, 43, 0, 512)
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
print(f"{os.path.basename(os.environ.get('FRR_LIBRARY', 'default'))}: mismatches={bad} rate={M / ms * 1e3:.3e} cand/s", flush=True)
