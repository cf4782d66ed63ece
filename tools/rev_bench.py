"""Generator throughput: thread-per-candidate reverse-bitset kernel
(frr_rev_bits, checksum only) vs the draw-arithmetic microbenchmark."""
import ctypes
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2501_07642_b200 import _native as N  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 1e3)
    return best


def main():
    dev = N.device()
    sink = torch.zeros(1, dtype=torch.int64, device=dev)
    res = {}
    for n, t, cnt in [(1000, 500, 1 << 24), (2000, 1000, 1 << 23), (5000, 2500, 1 << 21)]:
        s = timed(lambda: N.call("frr_rev_bits", ctypes.c_uint64(42), ctypes.c_uint64(0), cnt, n, t, None,
                                 N.ptr(sink), N.stream_ptr()))
        res[f"rev_{n}_{t}"] = {"cand_per_s": cnt / s, "draws_per_s": cnt * t / s}
    tot = ctypes.c_int64()
    s = timed(lambda: N.call("frr_microbench_draws", 4096, N.ptr(sink), ctypes.byref(tot), N.stream_ptr()))
    res["microbench_draws_per_s"] = tot.value / s
    print(json.dumps(res))


if __name__ == "__main__":
    main()
