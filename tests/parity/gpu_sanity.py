"""Quick on-GPU diagnosis of every libfrr entry point against the C oracle.
Prints one line per check; never raises (so one failure does not hide the
others).  Usage: python tests/parity/gpu_sanity.py"""

import os
import sys
import time
import traceback

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import oracle as O  # noqa: E402
import torch  # noqa: E402

import paper_2501_07642_b200 as frr  # noqa: E402
from paper_2501_07642_b200 import _native as N  # noqa: E402


RESULTS = []


def check(name, fn):
    t0 = time.time()
    try:
        ok, info = fn()
        torch.cuda.synchronize()
        print(f"[{'PASS' if ok else 'FAIL'}] {name}: {info} ({time.time() - t0:.2f}s)", flush=True)
        RESULTS.append(ok)
    except Exception as exc:  # noqa: BLE001
        print(f"[ERROR] {name}: {exc!r}", flush=True)
        RESULTS.append(False)
        traceback.print_exc()


def selftest(variant, K=128, N_=64):
    rng = np.random.default_rng(0)
    A = (rng.random((128, K)) < 0.5).astype(np.int8)
    B = rng.integers(-128, 128, size=(N_, K), dtype=np.int64).astype(np.int8)
    want = A.astype(np.int64) @ B.astype(np.int64).T
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    D = torch.zeros((128, N_), dtype=torch.int32, device="cuda")
    N.call("frr_selftest_mma_i8", N.ptr(dA), N.ptr(dB), K, N_, N.ptr(D), variant, N.stream_ptr())
    got = D.cpu().numpy().astype(np.int64)
    bad = int((got != want).sum())
    return bad == 0, f"variant {variant} K={K} N={N_}: {bad} mismatches"


def regen(n, t, seed=0xDEADBEEF, m=257):
    rng = np.random.default_rng(n)
    draws = np.concatenate([np.array([0, 1, 2**40, 2**64 - 1], dtype=np.uint64),
                            rng.integers(0, 2**63, size=m, dtype=np.int64).astype(np.uint64)])
    got = frr.batch_assignments(seed, draws, n, t)
    want = O.c_batch_assign(seed, draws, n, t)
    return np.array_equal(got, want), f"n={n} t={t} rows={draws.shape[0]}"


def mc_stats(n, d, t, M, path, mode="exact"):
    os.environ["FRR_MC_PATH"] = path
    X = np.random.default_rng(2).standard_normal((n, d))
    design = frr.DesignSpec(n, t, accept_prob=1.0, max_draws=M, batch_size=M, root_seed=42, precision_mode=mode)
    prec = frr.precompute_precision(X, mode)
    st = frr.generation.mc_stats_device(prec._kernel, design, 0, M).cpu().numpy()
    bal = O.balance_setup(X, O.precision(X, mode))
    want = O.c_mc_stats(bal, t, 42, 0, M)
    bad = int((st.view(np.uint64) != want.view(np.uint64)).sum())
    os.environ["FRR_MC_PATH"] = "auto"
    rel = float(np.max(np.abs(st - want) / np.maximum(np.abs(want), 1e-300)))
    return bad == 0, f"{path} n={n} d={d} M={M}: {bad} bit mismatches, max rel {rel:.2e}"


def exact(n, t, d):
    X = np.random.default_rng(n).standard_normal((n, d))
    import math

    M = math.comb(n, t)
    design = frr.DesignSpec(n, t, accept_prob=0.01, mode="exact", enumeration_cap=10**10)
    prec = frr.precompute_precision(X, "exact")
    st = frr.generation.exact_stats_device(prec._kernel, design, 0, M).cpu().numpy()
    bal = O.balance_setup(X, O.precision(X, "exact"))
    want = O.c_exact_stats(bal, t, 0, M)
    bad = int((st.view(np.uint64) != want.view(np.uint64)).sum())
    return bad == 0, f"exact n={n} t={t} d={d} M={M}: {bad} mismatches"


def select(M, p, ties):
    rng = np.random.default_rng(7)
    st = np.round(rng.random(M) * (4 if ties else 1e9)) / 7.0
    acc, thr = frr.generation._select(st, p)
    a2, t2 = O.c_select(st, p)
    return np.array_equal(acc, a2) and thr == t2, f"M={M} p={p} ties={ties} k={a2.shape[0]}"


def c1_pool():
    X = np.random.default_rng(1).standard_normal((20, 5))
    pool = frr.enumerate_exact(X, frr.DesignSpec(20, 10, accept_prob=0.01, mode="exact", batch_size=10_000))
    g = np.load(os.path.join(ROOT, "tests/golden/pools.npz"))
    ok = np.array_equal(pool.accepted_indices, g["c1_acc"]) and np.array_equal(pool.stats, g["c1_stats"])
    rng = np.random.default_rng(1)
    rng.standard_normal((20, 5))
    obs = pool.assignments[0]
    y = X @ rng.standard_normal(5) + 1.0 * obs + 0.5 * rng.standard_normal(20)
    res = frr.randomization_test(obs, y, pool, find_fi=True, alpha=0.05)
    ok2 = res.p_value == float(g["c1_p"]) and res.fi == tuple(g["c1_fi"]) and res.tau_obs == float(g["c1_tau"])
    return ok and ok2, f"pool {ok}, test {ok2}: p={res.p_value} fi={res.fi}"


def t5k():
    g = np.load(os.path.join(ROOT, "tests/golden/inference.npz"))
    W0 = frr.batch_assignments(5, np.array([0], dtype=np.uint64), 5000, 2500)[0]
    keys = np.column_stack([np.full(300, 5, dtype=np.uint64), 997 * np.arange(300, dtype=np.uint64)])
    pool = frr.RandomizationPool(
        design=frr.DesignSpec(5000, 2500, accept_prob=1.0, max_draws=300 * 997, batch_size=997, root_seed=5),
        stats=np.zeros(300), threshold_value=0.0, n_candidates=300 * 997, accepted_indices=997 * np.arange(300),
        keys=keys)
    res = frr.randomization_test(W0, g["t5k_y"], pool, find_fi=True, alpha=0.05)
    ok = (np.array_equal(res.stat_distribution, g["t5k_dist"]) and res.p_value == float(g["t5k_pv"])
          and res.fi == tuple(g["t5k_fi"]))
    return ok, f"p={res.p_value} fi={res.fi}"


def bench_mc(n=1000, d=64, t=500, M=1 << 22):
    X = np.random.default_rng(2).standard_normal((n, d))
    design = frr.DesignSpec(n, t, accept_prob=1e-3, max_draws=M, batch_size=M, root_seed=42)
    prec = frr.precompute_precision(X, "exact")
    out = torch.empty(M, dtype=torch.float64, device="cuda")
    res = []
    for path in ("tensor_core", "cuda_core"):
        os.environ["FRR_MC_PATH"] = path
        frr.generation.mc_stats_device(prec._kernel, design, 0, 1 << 16, out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        frr.generation.mc_stats_device(prec._kernel, design, 0, M, out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        res.append(f"{path}: {M / ms * 1e3:.3e} cand/s")
    os.environ["FRR_MC_PATH"] = "auto"
    return True, "; ".join(res)


if __name__ == "__main__":
    print(torch.cuda.get_device_name(0), flush=True)
    check("mma selftest v0", lambda: selftest(0))
    check("mma selftest v0 K=256 N=192", lambda: selftest(0, 256, 192))
    check("mma selftest A-in-TMEM K=128 N=64", lambda: selftest(2, 128, 64))
    check("mma selftest A-in-TMEM K=256 N=192", lambda: selftest(2, 256, 192))
    for n, t in [(2, 1), (10, 7), (33, 16), (1000, 500), (5000, 2500)]:
        check(f"regen {n},{t}", lambda n=n, t=t: regen(n, t))
    check("mc small 20x5", lambda: mc_stats(20, 5, 10, 20000, "cuda_core"))
    check("mc small 1000x8", lambda: mc_stats(1000, 8, 500, 4096, "cuda_core"))
    check("mc generic 30x40", lambda: mc_stats(30, 40, 15, 2000, "cuda_core", "ridge"))
    check("mc tc 30x40", lambda: mc_stats(30, 40, 15, 2000, "tensor_core", "ridge"))
    check("mc tc 1000x64", lambda: mc_stats(1000, 64, 500, 4096, "tensor_core"))
    check("mc nt 2000x1024", lambda: mc_stats(2000, 1024, 1000, 2048, "tensor_core", "ridge"))
    check("mc nt 300x200", lambda: mc_stats(300, 200, 150, 3000, "tensor_core", "ridge"))
    check("mc nt 1000x1001", lambda: mc_stats(1000, 1001, 17, 1000, "tensor_core", "ridge"))
    check("exact 20/10/5", lambda: exact(20, 10, 5))
    check("exact 26/13/5", lambda: exact(26, 13, 5))
    check("exact 24/12/20", lambda: exact(24, 12, 20))
    check("select ties", lambda: select(1_000_003, 0.01, True))
    check("select", lambda: select(3_000_000, 1e-3, False))
    check("C1 pool + test", c1_pool)
    check("t5k test path", t5k)
    check("bench mc 1000x64", bench_mc)
    print(f"SUMMARY: {sum(RESULTS)}/{len(RESULTS)} passed", flush=True)
