"""Pass-1 rates of the Monte Carlo tensor-core kernels for the C2 and C3
shapes (run twice: FRR_TC_FORCE_NT=0/1 routes C2 through the single-pass or
the N-tiled kernel), with a bit-exact check of a prefix against the oracle."""
import json
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

os.environ["FRR_MC_PATH"] = "tensor_core"
res = {"force_nt": os.environ.get("FRR_TC_FORCE_NT", "0")}
for name, n, t, d, mode, M, seed in [("c2", 1000, 500, 64, "exact", 1 << 24, 42),
                                     ("c3", 2000, 1000, 1024, "ridge", 1 << 21, 43)]:
    if len(sys.argv) > 1 and name not in sys.argv[1:]:
        continue
    X = np.random.default_rng(2 if name == "c2" else 3).standard_normal((n, d))
    prec = frr.precompute_precision(X, mode)
    kern = prec._kernel
    design = frr.DesignSpec(n, t, accept_prob=1e-3, max_draws=M, batch_size=10_000, root_seed=seed,
                            precision_mode=mode)
    out = torch.empty(M, dtype=torch.float64, device="cuda")
    G.mc_stats_device(kern, design, 0, M, out)
    torch.cuda.synchronize()
    chk = 4096
    want = O.c_mc_stats(O.balance_setup(X, prec.inverse), t, seed, 0, chk)
    got = out[:chk].cpu().numpy()
    mism = int((got.view(np.uint64) != want.view(np.uint64)).sum())
    best = 0.0
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        G.mc_stats_device(kern, design, 0, M, out)
        b.record()
        torch.cuda.synchronize()
        best = max(best, M / (a.elapsed_time(b) / 1e3))
    res[name] = {"cand_per_s": best, "prefix_mismatches": mism, "tc_kernel": int(kern.tc_plan()[0])}
print(json.dumps(res))
