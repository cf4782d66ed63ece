"""Where the C4 host-transfer time goes: raw pinned DMA rate, the host copy
out of pinned memory into a fresh numpy array (first-touch page faults) vs
into an already-touched one, and the repo's to_host_many, on the 117 MB C4
result shape.  Prints one line per probe (best of 5, ms)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_07642_b200 import _native as N  # noqa: E402

M = 2333606
dev = torch.device("cuda")
rows = torch.randint(0, 2, (M, 34), dtype=torch.int8, device=dev)
idx = torch.arange(M, dtype=torch.int64, device=dev)
st = torch.rand(M, dtype=torch.float64, device=dev)
nbytes = rows.numel() + idx.numel() * 8 + st.numel() * 8
pin = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
flat = torch.cat([rows.reshape(-1).view(torch.uint8), idx.view(torch.uint8), st.view(torch.uint8)])


def best(f, reps=5):
    f()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    return min(ts) * 1e3


def dma():
    pin.copy_(flat, non_blocking=True)
    torch.cuda.synchronize()


touched = np.ones(nbytes, np.uint8)


def host_fresh():
    out = np.empty(nbytes, np.uint8)
    np.copyto(out, pin.numpy())


def host_touched():
    np.copyto(touched, pin.numpy())


def fault_only():
    out = np.empty(nbytes, np.uint8)
    out[::4096] = 1


def repo():
    N.to_host_many(idx, st, rows)


thp = open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip() if os.path.exists(
    "/sys/kernel/mm/transparent_hugepage/enabled") else "?"
print(f"bytes {nbytes} cpus {os.cpu_count()} thp [{thp}]")
for name, f in [("dma_pinned", dma), ("host_copy_fresh", host_fresh), ("host_copy_touched", host_touched),
                ("first_touch_only", fault_only), ("to_host_many", repo)]:
    ms = best(f)
    print(f"{name:20s} {ms:7.2f} ms  {nbytes / ms / 1e6:6.1f} GB/s")
