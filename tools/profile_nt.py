"""One C3-shape tensor-core launch (N-tiled kernel) for ncu."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2501_07642_b200 as frr  # noqa: E402
from paper_2501_07642_b200 import generation as G  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
X = np.random.default_rng(3).standard_normal((2000, 1024))
design = frr.DesignSpec(2000, 1000, accept_prob=1e-4, max_draws=M, batch_size=min(M, 10_000), root_seed=43,
                        precision_mode="ridge")
kern = frr.precompute_precision(X, "ridge")._kernel
out = torch.empty(M, dtype=torch.float64, device="cuda")
for _ in range(2):
    G.mc_stats_device(kern, design, 0, M, out)
torch.cuda.synchronize()
print("ok", float(out[:4].sum()))
