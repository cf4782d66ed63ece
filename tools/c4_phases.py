"""Host/device phase breakdown of the C4 public-API call (exact n=34, t=17,
d=5, p=1e-3): pass 1, select, accepted-row regeneration, pool assembly."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2501_07642_b200 as frr  # noqa: E402
from paper_2501_07642_b200 import generation as G  # noqa: E402

X = np.random.default_rng(4).standard_normal((34, 5))
design = frr.DesignSpec(34, 17, accept_prob=1e-3, mode="exact", enumeration_cap=3 * 10**9)
marks = []


def wrap(mod, name):
    f = getattr(mod, name)

    def g(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize()
        marks.append((name, time.perf_counter() - t0))
        return r
    setattr(mod, name, g)


from paper_2501_07642_b200 import _native as NAT  # noqa: E402
from paper_2501_07642_b200 import _select as SEL  # noqa: E402

for nm in ["_select_device", "exact_rows_device", "_narrow_sample", "_narrow_filter", "_split_tables",
           "precompute_precision"]:
    wrap(G, nm)
for nm in ["bound_from_sample", "_select_full"]:
    wrap(SEL, nm)
wrap(NAT, "to_host")
wrap(G._Pass1, "__init__")
for it in range(3):
    marks.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pool = frr.generate_pool(X, design)
    torch.cuda.synchronize()
    tot = time.perf_counter() - t0
    print(f"total {tot * 1e3:.1f} ms", " ".join(f"{n}={s * 1e3:.1f}" for n, s in marks), pool.n_accepted)
import cProfile  # noqa: E402
import pstats  # noqa: E402

pr = cProfile.Profile()
pr.enable()
pool = frr.generate_pool(X, design)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
