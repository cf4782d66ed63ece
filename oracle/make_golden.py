"""Generate tests/golden/*.npz by importing the REFERENCE fastrr package.

Run in the build container only (it reads /root/reference, which does not
exist on the GPU box):

    OPENBLAS_NUM_THREADS=1 python oracle/make_golden.py

The fixtures pin the oracle (tests/test_oracle_golden.py) and the CUDA
product (tests/test_gpu_*.py) to the reference's own outputs.  Covariate
matrices are not stored: they are regenerated from numpy default_rng seeds
(deterministic for a fixed numpy), and their quantised integer forms are
pinned by hash.
"""

from __future__ import annotations

import hashlib
import os
import sys
import warnings

import numpy as np

REF = os.environ.get("FASTRR_REFERENCE_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)

import fastrr  # noqa: E402
from fastrr import balance as rb  # noqa: E402
from fastrr import generation as rg  # noqa: E402
from fastrr import inference as ri  # noqa: E402
from fastrr import keys as rk  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
M64 = (1 << 64) - 1


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def gen_keys():
    cases = [(2, 1), (5, 2), (10, 7), (33, 16), (64, 1), (12, 5), (20, 10), (1000, 500), (5000, 2500)]
    seeds = [0, 0xDEADBEEF, M64, 7]
    fixed = [0, 1, 2, 5, 100, 10**9, 2**40, M64]
    rng = np.random.default_rng(2024)
    rnd = rng.integers(0, 2**63, size=24, dtype=np.int64).astype(np.uint64)
    draws = np.concatenate([np.array(fixed, dtype=np.uint64), rnd, rnd * np.uint64(2) + np.uint64(1)])
    out = {"draws": draws, "cases": np.array(cases, dtype=np.int64),
           "seeds": np.array(seeds, dtype=np.uint64)}
    for n, t in cases:
        for si, s in enumerate(seeds):
            W = rk.batch_assignments(s, draws, n, t)
            out[f"bits_{n}_{t}_{si}"] = np.packbits(W.astype(np.uint8), axis=1, bitorder="little")
    # scalar path equals batch path (keys.py:138-159)
    a = rk.assignment_from_key(rk.AssignmentKey(7, 0), 20, 10)
    out["key7_0_20_10"] = np.flatnonzero(a.bits)
    out["state_samples"] = np.array(
        [[s, m, rk.derive_state(rk.AssignmentKey(s, m))] for s, m in
         [(0, 0), (7, 0), (7, 1), (12345, 999), (M64, M64), (0xDEADBEEF, 2**40)]], dtype=np.uint64)
    out["mix_samples"] = np.array([[z, rk.mix64(z)] for z in [0, 1, rk.GOLDEN, 2**63, M64]],
                                  dtype=np.uint64)
    np.savez_compressed(os.path.join(OUT, "keys.npz"), **out)


BAL_SHAPES = [  # (seed, n, d, mode, t, nkeys)
    (1, 20, 5, "exact", 10, 200),
    (2, 1000, 64, "exact", 500, 200),
    (4, 34, 5, "exact", 17, 200),
    (100, 12, 3, "exact", 6, 200),
    (108, 30, 40, "ridge", 15, 200),
    (10, 16, 3, "diagonal", 5, 200),
    (3, 100, 600, "ridge", 50, 64),
]


def gen_balance():
    out = {}
    for seed, n, d, mode, t, nk in BAL_SHAPES:
        X = np.random.default_rng(seed).standard_normal((n, d))
        prec = rb.precompute_precision(X, mode)
        kern = prec._kernel
        tag = f"{seed}_{n}_{d}_{mode}"
        out[f"zq_sha_{tag}"] = np.array(sha(kern._zq))
        out[f"inv_scale_sq_{tag}"] = np.array(kern._inv_scale_sq)
        W = rk.batch_assignments(seed, np.arange(nk, dtype=np.uint64), n, t)
        out[f"stats_{tag}"] = kern.stats(W, t)
        # mixed treated counts through batch_balance (balance.py:248-250)
        W2 = np.zeros((8, n), dtype=np.int8)
        for i in range(8):
            W2[i, : 1 + (i * (n - 2)) // 7] = 1
        out[f"mixed_{tag}"] = rb.batch_balance(X, prec, W2)
        if d <= 64:
            out[f"zq_{tag}"] = kern._zq.astype(np.int64)
    X = np.array([[1.0], [2.0], [3.0], [4.0]])
    out["hand_2_4"] = np.array(rb.mahalanobis_stat(X, rb.precompute_precision(X, "exact"),
                                                   np.array([1, 1, 0, 0], dtype=np.int8)))
    np.savez_compressed(os.path.join(OUT, "balance.npz"), **out)


def gen_pools():
    out = {}
    # exact n=10, t=5, p=0.2 (reference test_generation.py:59-74 shape)
    X = np.random.default_rng(102).standard_normal((10, 3))
    p = rg.enumerate_exact(X, rg.DesignSpec(10, 5, accept_prob=0.2, mode="exact"))
    out["e10_acc"], out["e10_stats"], out["e10_thr"] = p.accepted_indices, p.stats, np.array(p.threshold_value)
    out["e10_rows"] = p.assignments
    # C1 recipe: exact n=20,t=10,d=5,p=0.01 then a test + FI
    rng = np.random.default_rng(1)
    X = rng.standard_normal((20, 5))
    pool = rg.enumerate_exact(X, rg.DesignSpec(20, 10, accept_prob=0.01, mode="exact", batch_size=10_000))
    obs = pool.assignments[0]
    y = X @ rng.standard_normal(5) + 1.0 * obs + 0.5 * rng.standard_normal(20)
    res = ri.randomization_test(obs, y, pool, find_fi=True, alpha=0.05)
    out.update(c1_acc=pool.accepted_indices, c1_stats=pool.stats, c1_thr=np.array(pool.threshold_value),
               c1_y=y, c1_p=np.array(res.p_value), c1_tau=np.array(res.tau_obs),
               c1_fi=np.array(res.fi), c1_dist=res.stat_distribution)
    # Monte Carlo pools
    cov12 = rb.CovariateMatrix(np.random.default_rng(100).standard_normal((12, 3)))
    mc = {
        "mc12a": (cov12, rg.DesignSpec(12, 6, accept_prob=0.05, max_draws=2000, batch_size=97, root_seed=21)),
        "mc12all": (cov12, rg.DesignSpec(12, 6, accept_prob=1.0, max_draws=2000, batch_size=2000, root_seed=21)),
        "mc12one": (cov12, rg.DesignSpec(12, 6, accept_prob=0.01, max_draws=100, batch_size=10, root_seed=9)),
        "mctie": (np.ones((10, 1)), rg.DesignSpec(10, 5, accept_prob=0.02, max_draws=100, batch_size=25,
                                                  precision_mode="diagonal", root_seed=3)),
        "mc20": (np.random.default_rng(105).standard_normal((20, 5)),
                 rg.DesignSpec(20, 10, accept_prob=0.01, max_draws=100_000, batch_size=20_000, root_seed=12345)),
        "mcridge": (np.random.default_rng(108).standard_normal((30, 40)),
                    rg.DesignSpec(30, 15, accept_prob=0.1, max_draws=2000, batch_size=500,
                                  precision_mode="ridge", root_seed=31)),
        "mc1000": (np.random.default_rng(2).standard_normal((1000, 64)),
                   rg.DesignSpec(1000, 500, accept_prob=1e-3, max_draws=20_000, batch_size=10_000, root_seed=42)),
    }
    for name, (Xm, design) in mc.items():
        pl = rg.monte_carlo_pool(Xm, design, workers=1)
        out[f"{name}_acc"], out[f"{name}_stats"] = pl.accepted_indices, pl.stats
        out[f"{name}_thr"] = np.array(pl.threshold_value)
    np.savez_compressed(os.path.join(OUT, "pools.npz"), **out)


def gen_inference():
    out = {}
    X = np.random.default_rng(200).standard_normal((8, 2))
    pool8 = rg.enumerate_exact(X, rg.DesignSpec(8, 4, accept_prob=1.0, mode="exact", precision_mode="ridge"))
    mat = pool8.assignments
    rng = np.random.default_rng(201)
    ys, obs_i, pv, taus, dists = [], [], [], [], []
    for _ in range(100):
        y = rng.standard_normal(8) * rng.uniform(0.1, 10)
        i = int(rng.integers(0, 70))
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            r = ri.randomization_pvalue(mat[i], y, pool8)
        ys.append(y), obs_i.append(i), pv.append(r.p_value), taus.append(r.tau_obs), dists.append(r.stat_distribution)
    out.update(p8_rows=mat, p8_y=np.array(ys), p8_obs=np.array(obs_i), p8_p=np.array(pv),
               p8_tau=np.array(taus), p8_dist=np.array(dists))
    # fiducial intervals on pool8
    fis, fys, fobs, falpha = [], [], [], []
    rng = np.random.default_rng(207)
    for k in range(12):
        i = int(rng.integers(0, 70))
        y = rng.standard_normal(8) * 0.8 + 1.5 * mat[i]
        alpha = [0.05, 0.1, 0.25][k % 3]
        fis.append(ri.fiducial_interval(mat[i], y, pool8, alpha=alpha))
        fys.append(y), fobs.append(i), falpha.append(alpha)
    out.update(fi8=np.array(fis), fi8_y=np.array(fys), fi8_obs=np.array(fobs), fi8_alpha=np.array(falpha))
    # n=5000 test path
    W = rk.batch_assignments(5, 997 * np.arange(300, dtype=np.uint64), 5000, 2500)
    y = 2.0 * np.random.default_rng(5).standard_normal(5000) + W[0]
    p_at, tau_obs, a = ri._pvalue_curve(W, W[0], y, 2500)
    b = ri._dim_rows(W, W[0].astype(np.float64), 2500)
    tgrid = np.linspace(tau_obs - 3.0, tau_obs + 3.0, 64)
    out.update(t5k_y=y, t5k_a=a, t5k_b=b, t5k_tau=np.array(tau_obs), t5k_grid=tgrid,
               t5k_p=np.array([p_at(float(g)) for g in tgrid]))
    # a keys pool at n=5000 through randomization_test(find_fi)
    stats = np.zeros(300)
    pool = rg.RandomizationPool(
        design=rg.DesignSpec(5000, 2500, accept_prob=1.0, max_draws=300 * 997, batch_size=997, root_seed=5),
        stats=stats, threshold_value=0.0, n_candidates=300 * 997,
        accepted_indices=997 * np.arange(300), keys=np.column_stack(
            [np.full(300, 5, dtype=np.uint64), 997 * np.arange(300, dtype=np.uint64)]))
    res = ri.randomization_test(W[0], y, pool, find_fi=True, alpha=0.05)
    out.update(t5k_pv=np.array(res.p_value), t5k_fi=np.array(res.fi), t5k_dist=res.stat_distribution)
    np.savez_compressed(os.path.join(OUT, "inference.npz"), **out)


def gen_pairwise():
    rng = np.random.default_rng(77)
    out = {}
    for n in [1, 3, 7, 8, 9, 15, 16, 17, 63, 64, 65, 127, 128, 129, 200, 255, 256, 257, 1000, 1024, 4099, 5000]:
        rows = 16 if n < 1000 else 4
        a = rng.standard_normal((rows, n)) * rng.uniform(1e-3, 1e3, size=(rows, 1))
        a[0, :] = -0.0
        out[f"x_{n}"] = a
        out[f"s_{n}"] = a.sum(axis=1)
    np.savez_compressed(os.path.join(OUT, "pairwise.npz"), **out)


def gen_sim():
    """Synthetic-input helpers (bench.py:101-154): keyed normals, simulate_data
    inputs (X, coefficients, noise streams), the cost model."""
    from fastrr import bench as B

    out = {}
    for seed, stream, count in [(0, 0, 1), (7, 0, 1000), (7, 2, 999), (123, 5, 4096)]:
        out[f"normals_{seed}_{stream}_{count}"] = B.normals_from_stream(seed, stream, count)
    cfg = B.SimConfig(n=20, k=5)
    X, obs, y = B.simulate_data(cfg, seed=3)
    out["sim_X"], out["sim_bits"], out["sim_y"] = X.values, np.asarray(obs.bits), y
    cfg2 = B.SimConfig(n=12, k=3, coef=np.array([1.0, -2.0, 0.5]), tau_true=2.0, noise_sd=0.1)
    X2, obs2, y2 = B.simulate_data(cfg2, seed=11)
    out["sim2_X"], out["sim2_bits"], out["sim2_y"] = X2.values, np.asarray(obs2.bits), y2
    out["speedup"] = np.array([B.estimate_speedup(B.CostModel(0.5, 0.01, 2e-6, 64, 400.0, 10**8)),
                               B.estimate_speedup(B.CostModel(0.0, 1.0, 1.0, 1, 1.0, 0))])
    np.savez_compressed(os.path.join(OUT, "sim.npz"), **out)


def _unmix64(z: int) -> int:
    """Inverse of keys.py:107-115 (xorshifts and odd multipliers are bijections)."""
    def unxorshift(y, s):
        x = y
        for _ in range(64 // s + 1):
            x = y ^ (x >> s)
        return x & M64
    z = unxorshift(z, 31)
    z = (z * pow(0x94D049BB133111EB, -1, 1 << 64)) & M64
    z = unxorshift(z, 27)
    z = (z * pow(0xBF58476D1CE4E5B9, -1, 1 << 64)) & M64
    return unxorshift(z, 30)


def crafted_seed(draw: int, step: int, u: int) -> int:
    """A root seed whose key (seed, draw) has stream output `u` at Fisher-Yates
    step `step` (no earlier rejection): state0 = s_step - (step+1) C with
    s_step = mix64^-1(u); seed = (mix64^-1(state0) - C) ^ (draw C)."""
    g = rk.GOLDEN
    s_step = _unmix64(u)
    state0 = (s_step - (step + 1) * g) & M64
    pre = _unmix64(state0)
    seed = ((pre - g) & M64) ^ ((draw * g) & M64)
    assert rk.derive_state(rk.AssignmentKey(seed, draw)) == state0
    assert rk.mix64((state0 + (step + 1) * g) & M64) == u
    return seed


def gen_rejection():
    """Keys whose stream hits the rejection zone of _bounded (keys.py:148-155)
    at a chosen step (u = 2^64 - 1: rejected for every non-power-of-two
    bound), or only sets the GPU's "hi(u) == 0xFFFFFFFF" flag without a
    rejection (u = 0xFFFFFFFF00000000); outputs from the reference."""
    draw = 12345
    cases = [  # (n, t, step, u)
        (1000, 500, 7, M64), (1000, 500, 0, M64), (1000, 500, 499, M64), (1000, 500, 300, 0xFFFFFFFF00000000),
        (20, 10, 3, M64), (5000, 2500, 2000, M64), (2000, 1000, 999, M64), (1056, 1055, 1000, M64),
        (34, 17, 16, M64)]
    out = {"cases": np.array([c[:3] for c in cases], dtype=np.int64), "draw": np.array(draw, dtype=np.uint64)}
    seeds = []
    for i, (n, t, step, u) in enumerate(cases):
        seed = crafted_seed(draw, step, u)
        seeds.append(seed)
        W = rk.batch_assignments(seed, np.array([draw, draw + 1, 0], dtype=np.uint64), n, t)
        assert np.array_equal(W[0], np.asarray(rk.assignment_from_key(rk.AssignmentKey(seed, draw), n, t).bits))
        out[f"bits_{i}"] = np.packbits(W.astype(np.uint8), axis=1, bitorder="little")
    out["seeds"] = np.array(seeds, dtype=np.uint64)
    np.savez_compressed(os.path.join(OUT, "rejection.npz"), **out)


def _file_bytes(path) -> np.ndarray:
    with open(path, "rb") as f:
        return np.frombuffer(f.read(), dtype=np.uint8)


def gen_poolio():
    """Pool CSV files written by the reference (generation.py:388-525): Monte
    Carlo pools in keys / full / both storage, streamed with out_path and
    written with write_pool, and exact pools with and without out_path; plus
    the reference's read_pool of each file."""
    import dataclasses
    import json
    import tempfile

    out = {}
    X = np.random.default_rng(301).standard_normal((40, 3))
    base = rg.DesignSpec(n_units=40, n_treated=20, accept_prob=0.01, max_draws=3000, batch_size=257,
                         root_seed=301, precision_mode="exact")
    Xe = np.random.default_rng(302).standard_normal((12, 3))
    ex = rg.DesignSpec(n_units=12, n_treated=6, accept_prob=0.05, mode="exact", batch_size=100)
    with tempfile.TemporaryDirectory() as d:
        for storage in ("keys", "full", "both"):
            design = dataclasses.replace(base, storage=storage)
            path = os.path.join(d, f"mc_{storage}_stream.csv")
            rg.generate_pool(X, design, workers=1, out_path=path)
            out[f"mc_{storage}_stream"] = _file_bytes(path)
            pool = rg.generate_pool(X, design, workers=1)
            path = os.path.join(d, f"mc_{storage}_write.csv")
            rg.write_pool(pool, path)
            out[f"mc_{storage}_write"] = _file_bytes(path)
        path = os.path.join(d, "exact_stream.csv")
        rg.generate_pool(Xe, ex, out_path=path)
        out["exact_stream"] = _file_bytes(path)
        pool = rg.generate_pool(Xe, ex)
        path = os.path.join(d, "exact_write.csv")
        rg.write_pool(pool, path)
        out["exact_write"] = _file_bytes(path)
        # what the reference's reader makes of each file
        for name in [k for k in out]:
            path = os.path.join(d, name + ".csv")
            with open(path, "wb") as f:
                f.write(out[name].tobytes())
            rp = rg.read_pool(path)
            out[f"read_{name}"] = np.frombuffer(json.dumps({
                "design": rp.design.to_json_dict(), "threshold": rp.threshold_value,
                "n_candidates": rp.n_candidates, "stats": [repr(float(v)) for v in rp.stats],
                "accepted": None if rp.accepted_indices is None else [int(v) for v in rp.accepted_indices],
                "keys": None if rp.keys is None else [[int(a), int(b)] for a, b in rp.keys],
                "assignments_sha": None if rp.assignments is None else sha(rp.assignments.astype(np.int8)),
            }, sort_keys=True).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(OUT, "poolio.npz"), **out)


def gen_sweep():
    """threshold_sweep rows of the reference (inference.py:279-312) with and
    without the fiducial interval, including a failing row (accept_prob 0 is
    an invalid design: row-level isolation)."""
    import json

    X = np.random.default_rng(311).standard_normal((30, 3))
    rng = np.random.default_rng(312)
    y = X @ rng.standard_normal(3) + 0.5 * rng.standard_normal(30)
    base = rg.DesignSpec(n_units=30, n_treated=15, accept_prob=0.1, max_draws=4000, batch_size=500,
                         root_seed=311, precision_mode="exact")
    probs = [0.5, 0.1, 0.0, 0.02, 0.001]
    out = {}
    for find_fi in (False, True):
        rows = ri.threshold_sweep(X, base, probs, y, find_fi=find_fi, alpha=0.1, workers=1)
        out[f"rows_fi{int(find_fi)}"] = np.frombuffer(json.dumps(
            [{k: (repr(v) if isinstance(v, float) else v) for k, v in r.items()} for r in rows]).encode(),
            dtype=np.uint8)
    exb = rg.DesignSpec(n_units=12, n_treated=6, accept_prob=0.1, mode="exact")
    Xe = np.random.default_rng(313).standard_normal((12, 3))
    ye = Xe[:, 0] + 0.3 * np.random.default_rng(314).standard_normal(12)
    rows = ri.threshold_sweep(Xe, exb, [0.5, 0.2, 0.05, 0.01], ye, find_fi=True, alpha=0.2)
    out["rows_exact"] = np.frombuffer(json.dumps(
        [{k: (repr(v) if isinstance(v, float) else v) for k, v in r.items()} for r in rows]).encode(),
        dtype=np.uint8)
    out["probs"] = np.array(probs)
    np.savez_compressed(os.path.join(OUT, "sweep.npz"), **out)


GENERATORS = {"pairwise": lambda: gen_pairwise(), "keys": lambda: gen_keys(), "balance": lambda: gen_balance(),
              "pools": lambda: gen_pools(), "inference": lambda: gen_inference(), "sim": lambda: gen_sim(),
              "rejection": lambda: gen_rejection(), "poolio": lambda: gen_poolio(), "sweep": lambda: gen_sweep()}

if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    print("reference fastrr", fastrr.__version__, "from", REF)
    for name in sys.argv[1:] or list(GENERATORS):
        GENERATORS[name]()
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))
