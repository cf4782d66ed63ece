"""Per-role wait accounting of a FRR_NT_TIMING=1 build on the C3 (default) or C2 shape.
    python tools/nt_waits.py tools/variants/libfrr_ntim.so [c2|c3]"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["FRR_LIBRARY"] = os.path.abspath(sys.argv[1])
import paper_2501_07642_b200 as frr  # noqa: E402
from paper_2501_07642_b200 import _native as N  # noqa: E402
from paper_2501_07642_b200 import generation as G  # noqa: E402

if len(sys.argv) > 2 and sys.argv[2] == "c2":  # C2 through the N-tiled kernel (FRR_TC_FORCE_NT=1)
    os.environ["FRR_TC_FORCE_NT"] = "1"
    os.environ["FRR_MC_PATH"] = "tensor_core"
    X = np.random.default_rng(2).standard_normal((1000, 64))
    design = frr.DesignSpec(1000, 500, accept_prob=1e-3, max_draws=10**8, batch_size=10_000, root_seed=42)
    kern = frr.precompute_precision(X, "exact")._kernel
    M = 1 << 22
else:
    X = np.random.default_rng(3).standard_normal((2000, 1024))
    design = frr.DesignSpec(2000, 1000, accept_prob=1e-4, max_draws=10**8, batch_size=10_000, root_seed=43,
                            precision_mode="ridge")
    kern = frr.precompute_precision(X, "ridge")._kernel
    M = 1 << 20
out = torch.empty(M, dtype=torch.float64, device="cuda")
G.mc_stats_device(kern, design, 0, M, out)
buf = (ctypes.c_ulonglong * 16)()
N.lib().frr_debug_nt_waits(buf)
G.mc_stats_device(kern, design, 0, M, out)
N.lib().frr_debug_nt_waits(buf)
w = list(buf)
names = {0: "FY bits_empty", 1: "EXP bits_full", 2: "EXP s_empty", 3: "EPI tm_full", 4: "TMA s_empty",
         5: "MMA tm_empty", 6: "MMA full", 8: "FY total", 9: "EXP total", 10: "EPI total", 11: "MMA total",
         12: "TMA total"}
role = {0: 8, 1: 9, 2: 9, 3: 10, 4: 12, 5: 11, 6: 11}
for k, nm in names.items():
    frac = f"{100 * w[k] / w[role[k]]:6.2f}% of role" if k in role and w[role[k]] else ""
    print(f"{nm:14s} {w[k]:>16d} {frac}")
