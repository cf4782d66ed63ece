"""One frr_rev_bits launch (thread-per-candidate generator alone) for ncu:
    python tools/profile_rev.py n t count"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2501_07642_b200 import _native as N  # noqa: E402

n, t, cnt = (int(v) for v in sys.argv[1:4])
sink = torch.zeros(1, dtype=torch.int64, device=N.device())
for _ in range(2):
    N.call("frr_rev_bits", ctypes.c_uint64(42), ctypes.c_uint64(0), cnt, n, t, None, N.ptr(sink), N.stream_ptr())
torch.cuda.synchronize()
print("ok")
