"""A/B timing of the C5 statistics path (frr_dim_mc_ws, n=5000, t=2500,
1e6 keys) and its generator alone (frr_rev_bits) for the library named by
FRR_LIBRARY; prints one JSON line with a checksum of a and b so variants can
be compared for equality.  Usage: FRR_LIBRARY=... python tools/c5_ab.py [tag]"""
import ctypes
import hashlib
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2501_07642_b200 import _native as N  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return best


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else os.environ.get("FRR_LIBRARY", "default")
    n, t, m = 5000, 2500, 10**6
    dev = N.device()
    y = torch.from_numpy(np.random.default_rng(5).standard_normal(n)).to(dev)
    draws = torch.from_numpy(np.random.default_rng(6).integers(0, 10**8, m, dtype=np.int64)).to(dev)
    obs = torch.zeros((n + 31) // 32, dtype=torch.int32, device=dev)
    a = torch.empty(m, dtype=torch.float64, device=dev)
    b = torch.empty(m, dtype=torch.float64, device=dev)
    match = torch.zeros(1, dtype=torch.int32, device=dev)
    ws_bytes = int(N.lib().frr_dim_mc_workspace_bytes(m, n))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)

    def dim():
        N.call("frr_dim_mc_ws", 5, N.ptr(draws), m, n, t, N.ptr(y), N.ptr(obs), N.ptr(a), N.ptr(b), N.ptr(match),
               N.ptr(ws), ws_bytes, N.stream_ptr())

    s_dim = timed(dim)
    h = hashlib.sha1(a.cpu().numpy().tobytes() + b.cpu().numpy().tobytes()).hexdigest()[:12]
    sink = torch.zeros(1, dtype=torch.int64, device=dev)
    cnt = 1 << 20
    s_rev = timed(lambda: N.call("frr_rev_bits", ctypes.c_uint64(42), ctypes.c_uint64(0), cnt, n, t, None,
                                 N.ptr(sink), N.stream_ptr()))
    print(json.dumps({"tag": tag, "dim_ws_keys_per_s": m / s_dim, "dim_ws_ms": s_dim * 1e3,
                      "rev_keys_per_s": cnt / s_rev, "checksum": h, "sink": int(sink.item())}))


if __name__ == "__main__":
    main()
