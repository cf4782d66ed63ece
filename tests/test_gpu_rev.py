"""Thread-per-candidate generator (reverse-bitset Fisher-Yates,
csrc/frr_revfy.cuh) against the C oracle and the reference's golden keys,
bit-exact.  The fused Monte Carlo pass-1 kernel runs the same device code."""

import ctypes

import numpy as np
import pytest

import oracle as O
from paper_2501_07642_b200 import _native as N

pytestmark = pytest.mark.gpu


def rev_bits(seed, lo, count, n, t):
    import torch

    dev = N.device()
    kw = (n + 31) // 32
    out = torch.empty((count, kw), dtype=torch.int32, device=dev)
    N.call("frr_rev_bits", ctypes.c_uint64(seed), ctypes.c_uint64(lo), count, n, t, N.ptr(out), None, N.stream_ptr())
    bits = out.cpu().numpy().view(np.uint32)
    # control bits -> treated rows
    ctl = np.unpackbits(bits.view(np.uint8), axis=1, count=n, bitorder="little").astype(np.int8)
    return (1 - ctl).astype(np.int8)


@pytest.mark.parametrize("n,t", [(2, 1), (3, 2), (17, 8), (32, 31), (33, 32), (64, 32), (100, 1), (100, 99),
                                 (1000, 500), (1024, 512), (2000, 1000), (4097, 2000), (5000, 2500)])
def test_rev_vs_oracle(n, t):
    seed = 0x9E3779B97F4A7C15 ^ (n * 131 + t)
    lo = (n * 1_000_003) % (1 << 40)
    m = 3000 if n <= 2000 else 700
    got = rev_bits(seed, lo, m, n, t)
    want = O.c_batch_assign(seed, np.arange(lo, lo + m, dtype=np.uint64), n, t)
    assert np.array_equal(got, want), (n, t)


def test_rev_draw_range_wraps():
    lo = (1 << 64) - 70
    got = rev_bits(5, lo, 200, 1000, 500)
    draws = (np.arange(200, dtype=np.uint64) + np.uint64(lo))
    assert np.array_equal(got, O.c_batch_assign(5, draws, 1000, 500))


@pytest.mark.parametrize("case", range(9))
def test_rev_rejection_keys_golden(golden, case):
    """Keys crafted to be rejected at a chosen step (or only flagged) take
    the exact warp fallback inside the thread-per-candidate kernel."""
    g = golden("rejection")
    n, t, _ = (int(v) for v in g["cases"][case])
    seed, draw = int(g["seeds"][case]), int(g["draw"])
    want = np.unpackbits(g[f"bits_{case}"], axis=1, count=n, bitorder="little").astype(np.int8)
    got = rev_bits(seed, draw, 2, n, t)
    assert np.array_equal(got, want[:2])
