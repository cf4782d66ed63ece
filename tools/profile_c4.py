"""One exact pass-1 launch on the C4 shape (n=34, t=17, d=5) for ncu."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2501_07642_b200 as frr  # noqa: E402
from paper_2501_07642_b200 import generation as G  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26
X = np.random.default_rng(4).standard_normal((34, 5))
design = frr.DesignSpec(34, 17, accept_prob=1e-3, mode="exact", enumeration_cap=3 * 10**9)
kern = frr.precompute_precision(X, "exact")._kernel
out = torch.empty(M, dtype=torch.float64, device="cuda")
for _ in range(2):
    G.exact_stats_device(kern, design, 0, M, out)
torch.cuda.synchronize()
print("ok")
