"""tcgen05 kind::i8 throughput of single-CTA (M=128) vs CTA-pair
(cta_group::2, M=256) MMA streams, A from shared memory or TMEM, zero
operands: is the pair form worth it for the C3 kernel's shape (N=192)?"""
import ctypes
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2501_07642_b200 import _native as N  # noqa: E402

res = {}
for fn in ("frr_microbench_mma_i8", "frr_microbench_mma_i8_pair"):
    for a_tmem in (0, 1):
        for n in (128, 192, 256):
            ops = ctypes.c_int64(0)
            best = 0.0
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                N.call(fn, n, a_tmem, 20000, ctypes.byref(ops), N.stream_ptr())
                e1.record()
                torch.cuda.synchronize()
                best = max(best, ops.value / (e0.elapsed_time(e1) / 1e3))
            tag = f"{'pair' if fn.endswith('pair') else 'single'}_N{n}_{'tmemA' if a_tmem else 'smemA'}"
            res[tag] = best / 1e12
            print(f"{tag}: {best / 1e12:.0f} TOP/s int8", flush=True)
print(json.dumps(res))
