"""The C5 statistics kernels (frr_dim_mc_ws: k_rev_bits + k_dim_bits; FRR_C5_SINGLE=1: k_dim_rev)
on the C5 shape (n=5000, t=2500, 2^18 keys), for ncu."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2501_07642_b200 as frr  # noqa: E402
from paper_2501_07642_b200 import _native as N  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
y = torch.from_numpy(np.random.default_rng(5).standard_normal(5000)).cuda()
draws = torch.arange(m, dtype=torch.int64, device="cuda") * 997
obs = torch.zeros(157, dtype=torch.int32, device="cuda")
a = torch.empty(m, dtype=torch.float64, device="cuda")
b = torch.empty(m, dtype=torch.float64, device="cuda")
match = torch.zeros(1, dtype=torch.int32, device="cuda")
ws_bytes = int(N.lib().frr_dim_mc_workspace_bytes(m, 5000))
ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
for _ in range(2):
    if os.environ.get("FRR_C5_SINGLE"):
        N.call("frr_dim_mc", 5, N.ptr(draws), m, 5000, 2500, N.ptr(y), N.ptr(obs), N.ptr(a), N.ptr(b), N.ptr(match),
               N.stream_ptr())
    else:
        N.call("frr_dim_mc_ws", 5, N.ptr(draws), m, 5000, 2500, N.ptr(y), N.ptr(obs), N.ptr(a), N.ptr(b),
               N.ptr(match), N.ptr(ws), ws_bytes, N.stream_ptr())
torch.cuda.synchronize()
print("ok")
# one 512-point tau grid over the m keys (k_tau_counts)
taus = torch.linspace(-1.0, 1.0, 512, dtype=torch.float64, device="cuda")
rhs = torch.full((512,), 0.5, dtype=torch.float64, device="cuda")
counts = torch.empty(512, dtype=torch.int64, device="cuda")
for _ in range(2):
    N.call("frr_tau_counts", N.ptr(a), N.ptr(b), m, N.ptr(taus), N.ptr(rhs), 512, N.ptr(counts), N.stream_ptr())
torch.cuda.synchronize()
print("ok tau")
