"""Read the per-role wait accounting of a FRR_MMA_TIMING=1 build (C2 shape).
    python tools/waits.py tools/variants/libfrr_tim.so [M]"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["FRR_LIBRARY"] = os.path.abspath(sys.argv[1])
os.environ["FRR_MC_PATH"] = "tensor_core"
import paper_2501_07642_b200 as frr  # noqa: E402
from paper_2501_07642_b200 import _native as N  # noqa: E402
from paper_2501_07642_b200 import generation as G  # noqa: E402

M = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 21
X = np.random.default_rng(2).standard_normal((1000, 64))
design = frr.DesignSpec(1000, 500, accept_prob=1e-3, max_draws=M, batch_size=10_000, root_seed=42)
kern = frr.precompute_precision(X, "exact")._kernel
out = torch.empty(M, dtype=torch.float64, device="cuda")
G.mc_stats_device(kern, design, 0, M, out)
buf = (ctypes.c_ulonglong * 16)()
N.lib().frr_debug_waits(buf)
G.mc_stats_device(kern, design, 0, M, out)
N.lib().frr_debug_waits(buf)
w = list(buf)
names = ["FY bits_empty", "tile bits_full", "tile a_empty", "tile tmem_full", "TMA b_empty", "MMA tmem_empty",
         "MMA a_full", "MMA b_full", "FY total", "tile total", "MMA total", "FY in warp_fy", "TMA total",
         "tile epilogue"]
tot = {0: 8, 11: 8, 1: 9, 2: 9, 3: 9, 13: 9, 5: 10, 6: 10, 7: 10}
for k, nm in enumerate(names):
    frac = f"{100 * w[k] / w[tot[k]]:6.2f}% of role" if k in tot and w[tot[k]] else ""
    print(f"{nm:16s} {w[k]:>18d} {frac}")
