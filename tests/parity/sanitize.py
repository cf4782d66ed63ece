"""Small invocations of every hot-path kernel family for compute-sanitizer
(memcheck / racecheck / synccheck), each checked against the oracle:

    compute-sanitizer --tool racecheck python tests/parity/sanitize.py [case ...]

cases: c1 (exact n=20 pool + test/FI), c2 (tensor-core Monte Carlo prefix,
n=1000 d=64, 2^13 draws), c3 (N-tiled tensor-core prefix, n=2000 d=1024,
1024 draws), exact26 (fused split enumeration + narrowing, n=26),
c5 (2000 keys at n=5000: k_rev_bits + k_dim_bits, and k_dim_rev),
rejection (crafted keys through the exact fallback of the generators)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402
import paper_2501_07642_b200 as frr  # noqa: E402


def c1():
    X = np.random.default_rng(1).standard_normal((20, 5))
    pool = frr.enumerate_exact(X, frr.DesignSpec(20, 10, accept_prob=0.01, mode="exact"))
    st = O.c_exact_stats(O.balance_setup(X, O.precision(X, "exact")), 10, 0, 184_756)
    acc, thr = O.c_select(st, 0.01)
    assert np.array_equal(pool.accepted_indices, acc) and pool.threshold_value == thr
    r = frr.randomization_test(pool.assignments[0], X[:, 0] + pool.assignments[0], pool, find_fi=True)
    assert 0 < r.p_value <= 1


def _mc(n, t, d, mode, m, seed, xs):
    X = np.random.default_rng(xs).standard_normal((n, d))
    design = frr.DesignSpec(n, t, accept_prob=0.01, max_draws=m, batch_size=min(m, 10_000), root_seed=seed,
                            precision_mode=mode)
    pool = frr.monte_carlo_pool(X, design)
    prec = frr.precompute_precision(X, mode)
    want = O.c_mc_stats(O.balance_setup(X, prec.inverse), t, seed, 0, m)
    acc, thr = O.c_select(want, 0.01)
    assert np.array_equal(pool.accepted_indices, acc) and pool.threshold_value == thr


def c2():
    _mc(1000, 500, 64, "exact", 1 << 13, 42, 2)


def c3():
    _mc(2000, 1000, 1024, "ridge", 1024, 43, 3)


def exact26():
    from paper_2501_07642_b200 import _select as S

    S.PREFILTER_MIN = 1 << 20  # the fused narrowing path at this size
    X = np.random.default_rng(26).standard_normal((26, 5))
    pool = frr.enumerate_exact(X, frr.DesignSpec(26, 13, accept_prob=1e-3, mode="exact"))
    st = O.c_exact_stats(O.balance_setup(X, O.precision(X, "exact")), 13, 0, 10_400_600)
    acc, thr = O.c_select(st, 1e-3)
    assert np.array_equal(pool.accepted_indices, acc) and pool.threshold_value == thr


def c5():
    import torch

    from paper_2501_07642_b200 import _native as N

    n, t, m = 5000, 2500, 2000
    draws = np.arange(m, dtype=np.uint64) * np.uint64(997)
    W = frr.batch_assignments(5, draws, n, t)
    want = O.c_batch_assign(5, draws, n, t)
    assert np.array_equal(W, want)
    y = np.random.default_rng(5).standard_normal(n) + W[0]
    pool = frr.RandomizationPool(design=frr.DesignSpec(n, t, accept_prob=1.0, max_draws=m, batch_size=m, root_seed=5),
                                 stats=np.zeros(m), threshold_value=0.0, n_candidates=m,
                                 accepted_indices=draws.astype(np.int64),
                                 keys=np.column_stack([np.full(m, 5, dtype=np.uint64), draws]))
    r = frr.randomization_test(W[0], y, pool, find_fi=True)  # frr_dim_mc_ws
    assert np.array_equal(r.stat_distribution, O.c_dim_rows(want, y, t))
    # the single-kernel path (frr_dim_mc)
    dev = N.device()
    yd = torch.from_numpy(y).to(dev)
    dd = torch.from_numpy(draws.view(np.int64)).to(dev)
    obs = torch.zeros((n + 31) // 32, dtype=torch.int32, device=dev)
    a = torch.empty(m, dtype=torch.float64, device=dev)
    b = torch.empty(m, dtype=torch.float64, device=dev)
    N.call("frr_dim_mc", 5, N.ptr(dd), m, n, t, N.ptr(yd), N.ptr(obs), N.ptr(a), N.ptr(b), None, N.stream_ptr())
    assert np.array_equal(a.cpu().numpy(), r.stat_distribution)


def rejection():
    g = np.load(os.path.join(ROOT, "tests", "golden", "rejection.npz"))
    for case in range(g["cases"].shape[0]):
        n, t, _ = (int(v) for v in g["cases"][case])
        draws = np.array([int(g["draw"]), int(g["draw"]) + 1, 0], dtype=np.uint64)
        want = np.unpackbits(g[f"bits_{case}"], axis=1, count=n, bitorder="little").astype(np.int8)
        assert np.array_equal(frr.batch_assignments(int(g["seeds"][case]), draws, n, t), want)


CASES = {"c1": c1, "c2": c2, "c3": c3, "exact26": exact26, "c5": c5, "rejection": rejection}

if __name__ == "__main__":
    for name in sys.argv[1:] or list(CASES):
        CASES[name]()
        print("ok", name, flush=True)
