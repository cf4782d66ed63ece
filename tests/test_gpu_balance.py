"""GPU balance statistics vs the reference's golden statistics and the C
oracle -- bit-exact on every path (CUDA-core small-d, generic, tcgen05)."""

import math
import os

import numpy as np
import pytest

import oracle as O
import paper_2501_07642_b200 as frr
from paper_2501_07642_b200 import _native as N
from paper_2501_07642_b200 import generation as G

pytestmark = pytest.mark.gpu

SHAPES = [(1, 20, 5, "exact", 10), (2, 1000, 64, "exact", 500), (4, 34, 5, "exact", 17),
          (100, 12, 3, "exact", 6), (108, 30, 40, "ridge", 15), (10, 16, 3, "diagonal", 5)]


def bits_equal(a, b):
    return np.array_equal(np.asarray(a, dtype=np.float64).view(np.uint64), np.asarray(b, dtype=np.float64).view(np.uint64))


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"{s[1]}x{s[2]}{s[3]}")
def test_golden_stats_rows_path(golden, shape):
    seed, n, d, mode, t = shape
    g = golden("balance")
    tag = f"{seed}_{n}_{d}_{mode}"
    X = np.random.default_rng(seed).standard_normal((n, d))
    prec = frr.precompute_precision(X, mode)
    want = g[f"stats_{tag}"]
    W = frr.batch_assignments(seed, np.arange(want.shape[0], dtype=np.uint64), n, t)
    assert bits_equal(frr.batch_balance(X, prec, W), want)
    assert bits_equal(frr.batch_balance(X, prec, _mixed(n)), g[f"mixed_{tag}"])


def _mixed(n):
    W2 = np.zeros((8, n), dtype=np.int8)
    for i in range(8):
        W2[i, : 1 + (i * (n - 2)) // 7] = 1
    return W2


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"{s[1]}x{s[2]}{s[3]}")
@pytest.mark.parametrize("path", ["cuda_core", "tensor_core", "auto"])
def test_golden_stats_mc_paths(golden, shape, path, monkeypatch):
    seed, n, d, mode, t = shape
    g = golden("balance")
    want = g[f"stats_{seed}_{n}_{d}_{mode}"]
    X = np.random.default_rng(seed).standard_normal((n, d))
    kern = frr.precompute_precision(X, mode)._kernel
    if path == "tensor_core" and d <= 16:
        pytest.skip("tensor-core path is for d > 16")
    monkeypatch.setenv("FRR_MC_PATH", path)
    design = frr.DesignSpec(n, t, accept_prob=1.0, max_draws=want.shape[0], batch_size=1, root_seed=seed,
                            precision_mode=mode)
    st = G.mc_stats_device(kern, design, 0, want.shape[0]).cpu().numpy()
    assert bits_equal(st, want)


def test_hand_value():
    X = np.array([[1.0], [2.0], [3.0], [4.0]])
    st = frr.mahalanobis_stat(X, frr.precompute_precision(X, "exact"), np.array([1, 1, 0, 0], dtype=np.int8))
    assert st == pytest.approx(2.4, rel=1e-9)


# n spans the int8-limb counts (7 limbs n<=16, 6 limbs, 5 limbs n>4096)
MC_CASES = [(16, 20, 8, "ridge"), (17, 24, 8, "ridge"), (64, 33, 30, "exact"), (300, 80, 150, "exact"),
            (1000, 64, 500, "exact"), (1000, 64, 1, "exact"), (1000, 64, 999, "exact"), (2000, 70, 1000, "exact"),
            (4500, 32, 2250, "exact"), (1000, 8, 500, "exact"), (5000, 3, 2500, "exact"), (200, 130, 100, "ridge"),
            (2000, 1024, 1000, "ridge"), (1000, 1001, 17, "ridge"), (129, 300, 64, "diagonal"),
            # N-tiled kernel corner cases: odd limb count of 8*Zq (L=7), d not a
            # multiple of 32, tiny t; n=8200 x d=96 fits neither tensor-core kernel
            (20, 100, 10, "ridge"), (8200, 96, 4100, "exact"), (3000, 333, 2, "ridge"),
            # single-pass kernel at large n: fewer generator warps / one bit buffer
            (5000, 64, 2500, "exact"), (3000, 40, 1500, "exact"), (12000, 24, 6000, "exact"),
            # N-tiled kernel at large n: one bit buffer, fewer generators
            (5000, 128, 2500, "exact"),
            # t = n - 1 with n a multiple of 32: padding steps re-read past the table
            (1056, 64, 1055, "exact"), (1056, 8, 1055, "exact"), (1056, 40, 1055, "ridge")]


@pytest.mark.parametrize("n,d,t,mode", MC_CASES)
@pytest.mark.parametrize("path", ["auto", "cuda_core"])
def test_mc_stats_vs_oracle(n, d, t, mode, path, monkeypatch):
    X = np.random.default_rng(n * 31 + d).standard_normal((n, d)) * np.linspace(0.5, 3.0, d)
    M = 3001 if n * max(d, 16) < 200_000 or path == "auto" else 300
    if d > 200:
        M = 1024 if path == "auto" else 64
    monkeypatch.setenv("FRR_MC_PATH", path)
    kern = frr.precompute_precision(X, mode)._kernel
    if path == "auto" and (n, d) in ((20, 100), (3000, 333), (8200, 96), (5000, 64), (3000, 40), (5000, 128)):
        want = {(20, 100): 2, (3000, 333): 2, (8200, 96): 0, (5000, 64): 1, (3000, 40): 1, (5000, 128): 2}[(n, d)]
        assert kern.tc_plan()[0] == want
        if (n, d) == (20, 100):
            assert kern.tc_plan()[1] == 7  # 8*Zq needs 7 limbs: 128-byte K stages
    design = frr.DesignSpec(n, t, accept_prob=1.0, max_draws=10**9, batch_size=1, root_seed=n + d + t,
                            precision_mode=mode)
    lo = 10**9 - M
    st = G.mc_stats_device(kern, design, lo, M).cpu().numpy()
    bal = O.Balance(kern._zq, kern._inv_scale_sq)
    assert bits_equal(st, O.c_mc_stats(bal, t, design.root_seed, lo, M))


EXACT_CASES = [(20, 10, 5), (34, 17, 5), (12, 6, 3), (26, 13, 16), (24, 12, 20), (64, 3, 4), (80, 2, 5), (18, 9, 1),
               # split enumeration corners: t near 0 / n, odd n, widths 4/8/16
               (25, 1, 4), (25, 24, 7), (31, 5, 8), (36, 30, 12), (35, 18, 6), (24, 23, 16)]


@pytest.mark.parametrize("n,t,d", EXACT_CASES)
@pytest.mark.parametrize("path", ["auto", "successor"])
def test_exact_stats_vs_oracle(n, t, d, path, monkeypatch):
    monkeypatch.setenv("FRR_EXACT_PATH", path)
    X = np.random.default_rng(n + d).standard_normal((n, d))
    kern = frr.precompute_precision(X, "ridge")._kernel
    total = math.comb(n, t)
    lo = max(0, total - 250_000) if total > 500_000 else 0
    design = frr.DesignSpec(n, t, accept_prob=1.0, mode="exact", enumeration_cap=10**12, precision_mode="ridge")
    st = G.exact_stats_device(kern, design, lo, total - lo).cpu().numpy()
    bal = O.Balance(kern._zq, kern._inv_scale_sq)
    assert bits_equal(st, O.c_exact_stats(bal, t, lo, total - lo))
    if total > 500_000:  # also a window in the middle of the enumeration (block boundaries)
        mid = total // 2 - 77_777
        st = G.exact_stats_device(kern, design, mid, 150_001).cpu().numpy()
        assert bits_equal(st, O.c_exact_stats(bal, t, mid, 150_001))


@pytest.mark.parametrize("K,Nn", [(32, 16), (128, 64), (256, 192), (512, 256)])
def test_tcgen05_selftest(K, Nn):
    import torch

    rng = np.random.default_rng(K + Nn)
    A = (rng.random((128, K)) < 0.5).astype(np.int8)
    B = rng.integers(-128, 128, size=(Nn, K)).astype(np.int8)
    D = torch.zeros((128, Nn), dtype=torch.int32, device="cuda")
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    N.call("frr_selftest_mma_i8", N.ptr(dA), N.ptr(dB), K, Nn, N.ptr(D), 0, N.stream_ptr())
    assert np.array_equal(D.cpu().numpy().astype(np.int64), A.astype(np.int64) @ B.astype(np.int64).T)


def test_tensor_core_path_is_used_for_c2_shape():
    X = np.random.default_rng(2).standard_normal((1000, 64))
    kern = frr.precompute_precision(X, "exact")._kernel
    os.environ.pop("FRR_MC_PATH", None)
    assert kern.wants_tensor_cores() and kern.n_limbs == 6


def test_integration_md_ctypes_stub():
    """The binding INTEGRATION.md shows a fastrr maintainer (raw ctypes over
    include/frr.h, no package code on the call path) gives the package's
    statistics bit for bit."""
    import ctypes

    import torch

    from paper_2501_07642_b200 import _native as N

    lib = ctypes.CDLL(N.load_library()._name)

    class frr_balance_t(ctypes.Structure):
        _fields_ = [("n", ctypes.c_int32), ("d", ctypes.c_int32), ("t", ctypes.c_int32),
                    ("n_limbs", ctypes.c_int32), ("zq", ctypes.c_void_p), ("colsum", ctypes.c_void_p),
                    ("cc", ctypes.c_void_p), ("limbs", ctypes.c_void_p),
                    ("g", ctypes.c_double), ("cst", ctypes.c_double)]

    lib.frr_mc_stats.argtypes = [ctypes.POINTER(frr_balance_t), ctypes.c_uint64, ctypes.c_uint64,
                                 ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
    lib.frr_last_error.restype = ctypes.c_char_p

    X = np.random.default_rng(7).standard_normal((300, 12))
    design = frr.DesignSpec(300, 150, accept_prob=0.01, max_draws=20_000, root_seed=99)
    kernel = frr.precompute_precision(X, "exact")._kernel
    t, n = design.n_treated, kernel.n_units
    nc = n - t
    zq = torch.from_numpy(kernel._zq.astype("int64")).cuda()
    colsum = torch.from_numpy(kernel._colsum.astype("int64")).cuda()
    cc = torch.from_numpy(kernel._colsum * (1.0 / nc)).cuda()
    bal = frr_balance_t(n, zq.shape[1], t, 0, zq.data_ptr(), colsum.data_ptr(), cc.data_ptr(), None,
                        1.0 / t + 1.0 / nc, (t * nc / n) * kernel._inv_scale_sq)
    out = torch.empty(design.max_draws, dtype=torch.float64, device="cuda")
    rc = lib.frr_mc_stats(ctypes.byref(bal), design.root_seed, 0, design.max_draws, out.data_ptr(),
                          torch.cuda.current_stream().cuda_stream)
    assert rc == 0, lib.frr_last_error()
    want = G.mc_stats_device(kernel, design, 0, design.max_draws).cpu().numpy()
    assert bits_equal(out.cpu().numpy(), want)


@pytest.mark.parametrize("case,d,path", [(0, 64, "auto"), (0, 64, "cuda_core"), (2, 8, "auto"), (3, 40, "auto"),
                                         (6, 100, "auto"), (7, 64, "auto"), (5, 24, "auto")])
def test_mc_stats_rejection_keys(golden, case, d, path, monkeypatch):
    """Pass-1 statistics of a draw range containing a key crafted to hit the
    rejection zone (tests/golden/rejection.npz) on every pass-1 kernel."""
    g = golden("rejection")
    n, t, _ = (int(v) for v in g["cases"][case])
    seed, draw = int(g["seeds"][case]), int(g["draw"])
    X = np.random.default_rng(n + d).standard_normal((n, d))
    monkeypatch.setenv("FRR_MC_PATH", path)
    kern = frr.precompute_precision(X, "ridge")._kernel
    design = frr.DesignSpec(n, t, accept_prob=1.0, max_draws=10**6, batch_size=1, root_seed=seed,
                            precision_mode="ridge")
    lo, M = draw - 200, 400
    st = G.mc_stats_device(kern, design, lo, M).cpu().numpy()
    bal = O.Balance(kern._zq, kern._inv_scale_sq)
    assert bits_equal(st, O.c_mc_stats(bal, t, seed, lo, M))
