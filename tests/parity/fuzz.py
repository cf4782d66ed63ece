"""Randomized parity sweep (test infrastructure): random designs through the
GPU kernels, every output compared bit for bit with the C oracle.

Each case draws a random shape and checks, for whatever kernel routes serve
it (tensor-core single pass / N-tiled / CUDA-core by FRR_MC_PATH):
  mc     Monte Carlo pass-1 statistics of a random draw window;
  exact  exact-enumeration statistics of a random rank window (small n);
  regen  key -> assignment regeneration of random draws;
  dim    the randomization-test statistic a of random keys (thread-per-key
         stream path, frr_dim_mc_ws) for a random outcome vector;
  select the exact acceptance select (sampled narrowing above 2^22
         statistics) on random statistics with ties and zeros.

    python tests/parity/fuzz.py [seconds] [seed] > fuzz.json
prints one JSON summary line (cases per kind, mismatching cases listed)."""
import json
import math
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
from paper_2501_07642_b200.inference import _PoolStats  # noqa: E402


def bits_equal(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def case_mc(rng, path):
    n = int(rng.choice([int(rng.integers(4, 64)), int(rng.integers(64, 1200)), int(rng.integers(1200, 6000))]))
    d = int(rng.choice([int(rng.integers(1, 17)), int(rng.integers(17, 130)), int(rng.integers(130, 600))]))
    t = int(rng.integers(1, n))
    mode = str(rng.choice(["exact", "ridge", "diagonal"])) if d < n - 1 else str(rng.choice(["ridge", "diagonal"]))
    X = rng.standard_normal((n, d)) * rng.uniform(0.1, 10.0, d)
    os.environ["FRR_MC_PATH"] = path
    kern = frr.precompute_precision(X, mode)._kernel
    seed = int(rng.integers(0, 2**63))
    M = int(max(64, min(4000, 2_000_000 // (n * max(d, 8)))))
    lo = int(rng.integers(0, 2**40))
    design = frr.DesignSpec(n, t, accept_prob=1.0, max_draws=lo + M, batch_size=1, root_seed=seed,
                            precision_mode=mode)
    st = G.mc_stats_device(kern, design, lo, M).cpu().numpy()
    bal = O.Balance(kern._zq, kern._inv_scale_sq)
    ok = bits_equal(st, O.c_mc_stats(bal, t, seed, lo, M))
    return ok, dict(n=n, d=d, t=t, mode=mode, path=path, route=list(kern.tc_plan()), seed=seed, lo=lo, M=M)


def case_exact(rng):
    n = int(rng.integers(6, 37))
    t = int(rng.integers(1, n))
    d = int(rng.integers(1, 24))
    X = rng.standard_normal((n, d))
    kern = frr.precompute_precision(X, "ridge")._kernel
    total = math.comb(n, t)
    cnt = int(min(total, 200_000))
    lo = int(rng.integers(0, total - cnt + 1))
    design = frr.DesignSpec(n, t, accept_prob=1.0, mode="exact", enumeration_cap=10**12, precision_mode="ridge")
    st = G.exact_stats_device(kern, design, lo, cnt).cpu().numpy()
    bal = O.Balance(kern._zq, kern._inv_scale_sq)
    ok = bits_equal(st, O.c_exact_stats(bal, t, lo, cnt))
    return ok, dict(n=n, t=t, d=d, lo=lo, count=cnt)


def case_regen(rng):
    n = int(rng.choice([int(rng.integers(2, 100)), int(rng.integers(100, 3000)), int(rng.integers(3000, 20000))]))
    t = int(rng.integers(1, n))
    seed = int(rng.integers(0, 2**64, dtype=np.uint64))
    m = int(max(8, min(2000, 2_000_000 // n)))
    draws = rng.integers(0, 2**63, m).astype(np.uint64)
    got = frr.batch_assignments(seed, draws, n, t)
    ok = np.array_equal(got, O.c_batch_assign(seed, draws, n, t))
    return ok, dict(n=n, t=t, seed=seed, m=m)


def case_dim(rng):
    n = int(rng.choice([int(rng.integers(8, 200)), int(rng.integers(200, 2000)), int(rng.integers(2000, 9000))]))
    t = int(rng.integers(1, n))
    seed = int(rng.integers(0, 2**63))
    m = int(max(32, min(3000, 3_000_000 // n)))
    keys = np.column_stack([np.full(m, seed, dtype=np.uint64), rng.integers(0, 2**62, m).astype(np.uint64)])
    pool = frr.RandomizationPool(
        design=frr.DesignSpec(n, t, accept_prob=1.0, max_draws=2**62, batch_size=1, root_seed=seed),
        stats=np.zeros(m), threshold_value=0.0, n_candidates=2**62, accepted_indices=keys[:, 1].astype(np.int64),
        keys=keys)
    W = O.c_batch_assign(seed, keys[:, 1], n, t)
    y = rng.standard_normal(n) * rng.uniform(0.1, 100.0) + W[0]
    ps = _PoolStats(pool, W[0], y)
    ok = bits_equal(ps.a_local.cpu().numpy(), O.c_dim_rows(W, y, t))
    return ok, dict(n=n, t=t, seed=seed, m=m)


def case_select(rng):
    M = int(rng.choice([int(rng.integers(1000, 200_000)), int(rng.integers(4_200_000, 7_000_000))]))
    p = float(rng.choice([1e-4, 1e-3, 1e-2, 0.05, float(rng.uniform(1e-5, 0.2))]))
    ties = bool(rng.integers(0, 2))
    st = np.round(rng.random(M) * (7 if ties else 1e12)) / 3.0
    st[: int(rng.integers(0, M // 5 + 1))] = 0.0
    st = rng.permutation(st)
    acc, thr = G._select(st, p)
    want, wthr = O.c_select(st, p)
    return bool(np.array_equal(acc, want) and thr == wthr), dict(M=M, p=p, ties=ties)


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 2026)
    t_end = time.time() + budget
    counts, bad, routes = {}, [], {}
    kinds = ["mc_auto", "mc_cuda_core", "exact", "regen", "dim", "select"]
    i = 0
    while time.time() < t_end:
        kind = kinds[i % len(kinds)]
        i += 1
        if kind == "mc_auto":
            ok, info = case_mc(rng, "auto")
        elif kind == "mc_cuda_core":
            ok, info = case_mc(rng, "cuda_core")
        elif kind == "exact":
            ok, info = case_exact(rng)
        elif kind == "regen":
            ok, info = case_regen(rng)
        elif kind == "dim":
            ok, info = case_dim(rng)
        else:
            ok, info = case_select(rng)
        counts[kind] = counts.get(kind, 0) + 1
        if kind.startswith("mc"):
            r = "cuda_core" if kind == "mc_cuda_core" else {0: "cuda_core", 1: "tcgen05 single", 2: "tcgen05 N-tiled"}[
                info["route"][0]]
            routes[r] = routes.get(r, 0) + 1
        if not ok:
            bad.append(dict(kind=kind, **info))
    os.environ.pop("FRR_MC_PATH", None)
    print(json.dumps({"cases": counts, "mc_routes": routes, "total": sum(counts.values()), "mismatching_cases": bad,
                      "seconds": budget}))


if __name__ == "__main__":
    main()
