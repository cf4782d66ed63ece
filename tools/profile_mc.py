"""One short tensor-core MC launch (C2 shape) for ncu: warm-up launch, then
the profiled launch.  Usage: python tools/profile_mc.py [M] [path]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2501_07642_b200 as frr  # noqa: E402
from paper_2501_07642_b200 import generation as G  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 21
os.environ["FRR_MC_PATH"] = sys.argv[2] if len(sys.argv) > 2 else "tensor_core"
X = np.random.default_rng(2).standard_normal((1000, 64))
design = frr.DesignSpec(1000, 500, accept_prob=1e-3, max_draws=M, batch_size=min(M, 10_000), root_seed=42)
kern = frr.precompute_precision(X, "exact")._kernel
out = torch.empty(M, dtype=torch.float64, device="cuda")
for _ in range(2):
    G.mc_stats_device(kern, design, 0, M, out)
torch.cuda.synchronize()
print("ok", float(out[:4].sum()))
