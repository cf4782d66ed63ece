"""Throughput of every BASELINE.json config on one GPU (device time, CUDA
events), plus the roofline figure of each config's dominant kernel.

    python tools/bench_configs.py [c1 c2 c3 c4 c5]

C3/C4 are measured on bounded samples of their candidate ranges (stated);
the rates are candidates (or keys) per second of the pass-1 kernel, plus the
full-pool wall time where the full job is run."""

import json
import math
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2501_07642_b200 as frr  # noqa: E402
from paper_2501_07642_b200 import generation as G  # noqa: E402
from paper_2501_07642_b200.inference import _PoolStats  # noqa: E402

PEAKS = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return best


def c1():
    rng = np.random.default_rng(1)
    X = rng.standard_normal((20, 5))
    design = frr.DesignSpec(20, 10, accept_prob=0.01, mode="exact", batch_size=10_000)
    beta, noise = rng.standard_normal(5), 0.5 * rng.standard_normal(20)

    def job():
        pool = frr.enumerate_exact(X, design)
        obs = pool.assignments[0]
        y = X @ beta + 1.0 * obs + noise
        return frr.randomization_test(obs, y, pool, find_fi=True)

    t0 = time.perf_counter()
    job()  # first call in the process: CUDA context, module load, allocator warm-up
    cold = time.perf_counter() - t0
    walls = []
    for _ in range(3):
        t0 = time.perf_counter()
        res = job()
        walls.append(time.perf_counter() - t0)
    wall = min(walls)
    kern = frr.precompute_precision(X, "exact")._kernel
    out = torch.empty(184_756, dtype=torch.float64, device="cuda")
    s = timed(lambda: G.exact_stats_device(kern, design, 0, 184_756, out))
    return {"config": "C1 exact n=20 t=10 d=5 p=0.01 + test/FI", "candidates": 184_756,
            "pass1_cand_per_s": 184_756 / s, "pass1_ms": s * 1e3, "api_wall_ms_pool_plus_test": wall * 1e3,
            "api_wall_ms_first_call": cold * 1e3,
            "p_value": res.p_value, "fi": res.fi}


def c2():
    X = np.random.default_rng(2).standard_normal((1000, 64))
    M = 10**8
    design = frr.DesignSpec(1000, 500, accept_prob=1e-3, max_draws=M, batch_size=10_000, root_seed=42)
    kern = frr.precompute_precision(X, "exact")._kernel
    out = torch.empty(M, dtype=torch.float64, device="cuda")
    s = timed(lambda: G.mc_stats_device(kern, design, 0, M, out), reps=2)
    tf = M * 2 * 1000 * 64 / s / 1e12
    return {"config": "C2 MC n=1000 t=500 d=64 1e8", "pass1_cand_per_s": M / s, "pass1_ms": s * 1e3,
            "tensor_TFLOPs_algorithmic": tf, "frac_of_bf16_sustained": tf / PEAKS.get("bf16_tflops_sustained", 1382.1)}


def c3(M=2_000_000):
    X = np.random.default_rng(3).standard_normal((2000, 1024))
    design = frr.DesignSpec(2000, 1000, accept_prob=1e-4, max_draws=10**8, batch_size=10_000, root_seed=43,
                            precision_mode="ridge")
    kern = frr.precompute_precision(X, "ridge")._kernel
    out = torch.empty(M, dtype=torch.float64, device="cuda")
    s = timed(lambda: G.mc_stats_device(kern, design, 0, M, out), reps=3)
    tf = M * 2 * 2000 * 1024 / s / 1e12
    kind, L = kern.tc_plan()
    kpad, dpad = (2000 + 127) // 128 * 128, (1024 + 31) // 32 * 32
    executed = M * 2 * kpad * L * dpad / s / 1e12  # int8 tensor ops actually issued
    peak = _mma_peak(192)
    return {"config": f"C3 MC n=2000 t=1000 d=1024 ridge (sample of {M} draws)", "pass1_cand_per_s": M / s,
            "tensor_TFLOPs_algorithmic": tf, "int8_TOPs_executed": executed, "limbs": L,
            "int8_peak_TOPs_measured": peak, "frac_of_measured_int8_peak": executed / peak,
            "peak_source": "frr_microbench_mma_i8(N=192, A in TMEM): the kernel's own MMA shape, back to back",
            "path": {1: "tcgen05 single", 2: "tcgen05 N-tiled"}.get(kind, "cuda_core")}


def _mma_peak(n, a_tmem=1):
    import ctypes

    from paper_2501_07642_b200 import _native as N

    ops = ctypes.c_int64(0)
    best = 0.0
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        N.call("frr_microbench_mma_i8", n, a_tmem, 20000, ctypes.byref(ops), N.stream_ptr())
        e1.record()
        torch.cuda.synchronize()
        best = max(best, ops.value / (e0.elapsed_time(e1) / 1e3))
    return best / 1e12


def c4(M=500_000_000):
    X = np.random.default_rng(4).standard_normal((34, 5))
    total = math.comb(34, 17)
    design = frr.DesignSpec(34, 17, accept_prob=1e-3, mode="exact", enumeration_cap=3 * 10**9)
    kern = frr.precompute_precision(X, "exact")._kernel
    out = torch.empty(M, dtype=torch.float64, device="cuda")
    s = timed(lambda: G.exact_stats_device(kern, design, 0, M, out), reps=2)
    gbs = M * 8 / s / 1e9
    torch.cuda.synchronize()
    del out
    torch.cuda.empty_cache()
    full = frr.DesignSpec(34, 17, accept_prob=1e-3, mode="exact", enumeration_cap=3 * 10**9)
    walls = {}
    for mode in ("0", "1"):  # unfused (18.7 GB statistics array + select), fused pass 1 + narrowing
        os.environ["FRR_EXACT_FUSED_SELECT"] = mode
        frr.enumerate_exact(X, full)  # first call: allocations enter torch's cache
        best = float("inf")
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            pool = frr.enumerate_exact(X, full)
            best = min(best, time.perf_counter() - t0)
        walls[mode] = best
        del pool
        torch.cuda.empty_cache()
    os.environ.pop("FRR_EXACT_FUSED_SELECT")
    pool = frr.enumerate_exact(X, full)
    wall = walls["1"]
    return {"config": "C4 exact n=34 t=17 d=5 p=1e-3 (2.33e9 ranks)", "pass1_sample": M,
            "pass1_cand_per_s": M / s, "stat_write_GBps": gbs, "frac_hbm": gbs / PEAKS["hbm_gbs"],
            "full_pool_wall_s": wall, "full_cand_per_s": total / wall,
            "full_pool_wall_s_unfused": walls["0"], "accepted": pool.n_accepted,
            "threshold": pool.threshold_value}


def c5(m=10**6):
    keys = np.column_stack([np.full(m, 5, dtype=np.uint64), 997 * np.arange(m, dtype=np.uint64)])
    pool = frr.RandomizationPool(
        design=frr.DesignSpec(5000, 2500, accept_prob=1.0, max_draws=m * 997, batch_size=997, root_seed=5),
        stats=np.zeros(m), threshold_value=0.0, n_candidates=m * 997, accepted_indices=997 * np.arange(m), keys=keys)
    X = np.random.default_rng(5).standard_normal((5000, 64))
    obs = frr.batch_assignments(5, np.array([0], dtype=np.uint64), 5000, 2500)[0]
    rng = np.random.default_rng(5)
    y = X @ rng.standard_normal(64) + 1.0 * obs + 0.5 * rng.standard_normal(5000)
    ps = [None]

    def stats():
        ps[0] = _PoolStats(pool, obs, y)

    s_keys = timed(stats, reps=5)
    p = ps[0]
    sd = float(np.std(p.a.cpu().numpy()))
    taus = np.linspace(p.tau_obs - 10 * sd, p.tau_obs + 10 * sd, 512)
    rhs = [abs(p.tau_obs - float(t) * p.b_obs) for t in taus]
    s_grid = timed(lambda: p.counts(taus, rhs), reps=3)
    frr.randomization_test(obs, y, pool, find_fi=True)  # first call: staging buffers, module loads
    t0 = time.perf_counter()
    res = frr.randomization_test(obs, y, pool, find_fi=True)
    wall = time.perf_counter() - t0
    return {"config": "C5 test+FI n=5000 t=2500, 1e6 keys, 512-tau grid", "keys_per_s": m / s_keys,
            "regen_plus_dim_ms": s_keys * 1e3,
            # algorithmic HBM bytes: 16 per key (a, b written); the grid reads them (16 per key per launch)
            "dim_hbm_GBps": 16 * m / s_keys / 1e9, "dim_frac_hbm": 16 * m / s_keys / 1e9 / PEAKS["hbm_gbs"],
            "dim_bound": "int issue / latency (generator + masked pairwise sums; a, b stay in L2)",
            "grid_key_tau_per_s": m * 512 / s_grid, "grid_ms": s_grid * 1e3,
            "grid_hbm_GBps": 16 * m / s_grid / 1e9,
            "randomization_test_find_fi_wall_s": wall, "p_value": res.p_value, "fi": res.fi}


if __name__ == "__main__":
    which = sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5"]
    print(torch.cuda.get_device_name(0), flush=True)
    for w in which:
        try:
            print(json.dumps(globals()[w]()), flush=True)
        except Exception as exc:  # noqa: BLE001
            print(json.dumps({"config": w, "error": repr(exc)}), flush=True)
