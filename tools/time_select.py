"""Wall time of select_k_smallest on 1e8 device statistics (C2 step's select)."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2501_07642_b200._select import DeviceSelectOps, LocalComm, select_k_smallest  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 10**8
g = torch.Generator(device="cuda").manual_seed(1)
st = torch.rand(M, dtype=torch.float64, device="cuda", generator=g) * 20
ops = DeviceSelectOps()
for pf in (True, False):
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        idx, val, thr = select_k_smallest(st, 0, M // 1000, ops, LocalComm(), prefilter=pf)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"prefilter={pf}: {dt * 1e3:.2f} ms, k={idx.numel()}")
import cProfile  # noqa: E402
import pstats  # noqa: E402

pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    select_k_smallest(st, 0, M // 1000, ops, LocalComm())
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
