"""The C2 step's select on 1e8 device statistics (narrowing + radix passes) for ncu."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2501_07642_b200._select import DeviceSelectOps, LocalComm, select_k_smallest  # noqa: E402

M = 10**8
g = torch.Generator(device="cuda").manual_seed(1)
st = torch.rand(M, dtype=torch.float64, device="cuda", generator=g) * 20
for _ in range(2):
    select_k_smallest(st, 0, M // 1000, DeviceSelectOps(), LocalComm())
torch.cuda.synchronize()
print("ok")
