"""Full-size parity runs: every statistic of the C2 workload
(1e8 Monte Carlo candidates), of C4 (2.33e9 exact ranks) and every C5 test
statistic (1e6 keys) from
the GPU path compared bit for bit with the C oracle (test infrastructure,
multi-threaded on the host), and the accepted pools compared with the
oracle's stable selection.

    python tests/parity/full_parity.py c2 [c4] [c5] > result.json"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402

import paper_2501_07642_b200 as frr  # noqa: E402
from paper_2501_07642_b200 import generation as G  # noqa: E402


def run(name, X, design, oracle_stats, chunk):
    t0 = time.perf_counter()
    pool = frr.generate_pool(X, design)
    t_pool = time.perf_counter() - t0
    kern = frr.precompute_precision(X, design.precision_mode)._kernel
    M = pool.n_candidates
    mism, first_bad = 0, None
    t0 = time.perf_counter()
    want_all = np.empty(M, dtype=np.float64)
    for lo in range(0, M, chunk):
        c = min(chunk, M - lo)
        gpu = (G.mc_stats_device if design.mode == "monte_carlo" else G.exact_stats_device)(kern, design, lo, c)
        got = gpu.cpu().numpy()
        want = oracle_stats(lo, c)
        want_all[lo:lo + c] = want
        bad = np.flatnonzero(got.view(np.uint64) != want.view(np.uint64))
        if bad.size and first_bad is None:
            first_bad = int(lo + bad[0])
        mism += int(bad.size)
    t_cmp = time.perf_counter() - t0
    acc, thr = O.c_select(want_all, design.accept_prob)
    return {"config": name, "candidates": M, "stat_mismatches": mism, "first_mismatch": first_bad,
            "accepted": int(pool.n_accepted), "accepted_equal": bool(np.array_equal(pool.accepted_indices, acc)),
            "accepted_stats_equal": bool(np.array_equal(pool.stats, want_all[acc])),
            "threshold_equal": pool.threshold_value == thr, "gpu_pool_s": t_pool, "oracle_compare_s": t_cmp}


def c2():
    X = np.random.default_rng(2).standard_normal((1000, 64))
    design = frr.DesignSpec(1000, 500, accept_prob=1e-3, max_draws=10**8, batch_size=10_000, root_seed=42)
    bal = O.balance_setup(X, O.precision(X, "exact"))
    return run("C2 full (1e8 MC draws)", X, design, lambda lo, c: O.c_mc_stats(bal, 500, 42, lo, c), 10**7)


def c4():
    X = np.random.default_rng(4).standard_normal((34, 5))
    design = frr.DesignSpec(34, 17, accept_prob=1e-3, mode="exact", enumeration_cap=3 * 10**9)
    bal = O.balance_setup(X, O.precision(X, "exact"))
    return run("C4 full (2.33e9 exact ranks)", X, design, lambda lo, c: O.c_exact_stats(bal, 17, lo, c), 2 * 10**8)


def c3():
    """C3 at full size (1e8 draws, n=2000, d=1024): the oracle cannot recompute
    all 1e8 statistics, so it recomputes every accepted one, the 2000 ranks
    around the threshold and 1e6 random draws; the pool must equal the
    selection over the GPU statistics."""
    X = np.random.default_rng(3).standard_normal((2000, 1024))
    M = 10**8
    design = frr.DesignSpec(2000, 1000, accept_prob=1e-4, max_draws=M, batch_size=10_000, root_seed=43,
                            precision_mode="ridge")
    t0 = time.perf_counter()
    pool = frr.generate_pool(X, design)
    t_pool = time.perf_counter() - t0
    kern = frr.precompute_precision(X, "ridge")._kernel
    st = G.mc_stats_device(kern, design, 0, M).cpu().numpy()
    k = G._accepted_count(1e-4, M)
    order = np.argsort(st, kind="stable")
    acc = np.sort(order[:k])
    rng = np.random.default_rng(31)
    idx = np.unique(np.concatenate([order[: k + 1000], rng.integers(0, M, size=1_000_000)]))
    bal = O.balance_setup(X, O.precision(X, "ridge"))
    t0 = time.perf_counter()
    want = np.empty(idx.shape[0], dtype=np.float64)
    for lo in range(0, idx.shape[0], 5000):
        rows = O.c_batch_assign(43, idx[lo:lo + 5000].astype(np.uint64), 2000, 1000)
        want[lo:lo + rows.shape[0]] = O.c_stats_rows(bal, rows, 1000)
    return {"config": "C3 full (1e8 MC draws, n=2000, d=1024)", "candidates": M, "checked": int(idx.shape[0]),
            "stat_mismatches": int(np.count_nonzero(st[idx].view(np.uint64) != want.view(np.uint64))),
            "accepted": int(pool.n_accepted), "accepted_equal": bool(np.array_equal(pool.accepted_indices, acc)),
            "accepted_stats_equal": bool(np.array_equal(pool.stats, st[acc])),
            "threshold_equal": bool(pool.threshold_value == st[order[k - 1]]), "gpu_pool_s": t_pool,
            "oracle_s": time.perf_counter() - t0}


def c5(m=10**6):
    """C5 test statistics of all 1e6 keys (n=5000): a = difference in means of
    every regenerated assignment, b from the popcounts, and the p-value, against
    the oracle's regeneration + numpy-order masked sums."""
    from paper_2501_07642_b200.inference import _PoolStats

    keys = np.column_stack([np.full(m, 5, dtype=np.uint64), 997 * np.arange(m, dtype=np.uint64)])
    pool = frr.RandomizationPool(
        design=frr.DesignSpec(5000, 2500, accept_prob=1.0, max_draws=m * 997, batch_size=997, root_seed=5),
        stats=np.zeros(m), threshold_value=0.0, n_candidates=m * 997, accepted_indices=997 * np.arange(m), keys=keys)
    X = np.random.default_rng(5).standard_normal((5000, 64))
    obs = frr.batch_assignments(5, np.array([0], dtype=np.uint64), 5000, 2500)[0]
    rng = np.random.default_rng(5)
    y = X @ rng.standard_normal(64) + 1.0 * obs + 0.5 * rng.standard_normal(5000)
    ps = _PoolStats(pool, obs, y)
    a = ps.a.cpu().numpy()
    res = frr.randomization_pvalue(obs, y, pool)
    want = np.empty(m, dtype=np.float64)
    t0 = time.perf_counter()
    for lo in range(0, m, 20_000):
        rows = O.c_batch_assign(5, keys[lo:lo + 20_000, 1], 5000, 2500)
        want[lo:lo + rows.shape[0]] = O.c_dim_rows(rows, y, 2500)
    tau_obs = float(O.c_dim_rows(np.asarray(obs, dtype=np.int8).reshape(1, -1), y, 2500)[0])
    p_want = float(np.count_nonzero(np.abs(want) >= abs(tau_obs))) / m
    return {"config": "C5 full (1e6 keys, n=5000)", "keys": m,
            "a_mismatches": int(np.count_nonzero(a.view(np.uint64) != want.view(np.uint64))),
            "tau_obs_equal": ps.tau_obs == tau_obs, "p_value": res.p_value, "p_value_equal": res.p_value == p_want,
            "oracle_s": time.perf_counter() - t0}


if __name__ == "__main__":
    for name in sys.argv[1:] or ["c2"]:
        print(json.dumps({"c2": c2, "c3": c3, "c4": c4, "c5": c5}[name]()), flush=True)
