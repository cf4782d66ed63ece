"""GPU randomization tests and fiducial intervals vs the reference's golden
p-values / intervals (bit-exact) and brute-force oracles."""

import dataclasses
import warnings

import numpy as np
import pytest

import oracle as O
import paper_2501_07642_b200 as frr
from paper_2501_07642_b200.errors import EmptyIntervalError, InvalidDesignError, UnsupportedStatisticError

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pool8(golden):
    X = np.random.default_rng(200).standard_normal((8, 2))
    pool = frr.enumerate_exact(X, frr.DesignSpec(8, 4, accept_prob=1.0, mode="exact", precision_mode="ridge"))
    assert np.array_equal(pool.assignments, golden("inference")["p8_rows"])
    return pool


def test_pvalues_golden(pool8, golden):
    g = golden("inference")
    rows = pool8.assignments
    for y, i, p, tau, dist in zip(g["p8_y"], g["p8_obs"], g["p8_p"], g["p8_tau"], g["p8_dist"]):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            res = frr.randomization_pvalue(rows[i], y, pool8)
        assert res.p_value == p and res.tau_obs == tau
        assert np.array_equal(res.stat_distribution, dist)
        assert res.obs_in_pool


def test_fi_golden(pool8, golden):
    g = golden("inference")
    rows = pool8.assignments
    for fi, y, i, alpha in zip(g["fi8"], g["fi8_y"], g["fi8_obs"], g["fi8_alpha"]):
        assert frr.fiducial_interval(rows[i], y, pool8, alpha=float(alpha)) == tuple(fi)


def test_c1_test_golden(golden):
    g = golden("pools")
    rng = np.random.default_rng(1)
    X = rng.standard_normal((20, 5))
    pool = frr.enumerate_exact(X, frr.DesignSpec(20, 10, accept_prob=0.01, mode="exact", batch_size=10_000))
    obs = pool.assignments[0]
    y = X @ rng.standard_normal(5) + 1.0 * obs + 0.5 * rng.standard_normal(20)
    assert np.array_equal(y, g["c1_y"])
    res = frr.randomization_test(obs, y, pool, find_fi=True, alpha=0.05)
    assert res.p_value == float(g["c1_p"]) == 0.022198159177043854
    assert res.tau_obs == float(g["c1_tau"])
    assert res.fi == (0.16286956452528453, 1.5386068617648494)
    assert np.array_equal(res.stat_distribution, g["c1_dist"])


def _t5k_pool(m=300):
    keys = np.column_stack([np.full(m, 5, dtype=np.uint64), 997 * np.arange(m, dtype=np.uint64)])
    return frr.RandomizationPool(
        design=frr.DesignSpec(5000, 2500, accept_prob=1.0, max_draws=m * 997, batch_size=997, root_seed=5),
        stats=np.zeros(m), threshold_value=0.0, n_candidates=m * 997, accepted_indices=997 * np.arange(m), keys=keys)


def test_keys_pool_n5000_golden(golden):
    g = golden("inference")
    pool = _t5k_pool()
    W0 = frr.batch_assignments(5, np.array([0], dtype=np.uint64), 5000, 2500)[0]
    res = frr.randomization_test(W0, g["t5k_y"], pool, find_fi=True, alpha=0.05)
    assert np.array_equal(res.stat_distribution, g["t5k_dist"])
    assert res.p_value == float(g["t5k_pv"]) and res.fi == tuple(g["t5k_fi"])
    # the same pool as explicit rows gives the identical test
    rows_pool = frr.RandomizationPool(design=pool.design, stats=pool.stats, threshold_value=0.0,
                                      n_candidates=pool.n_candidates, accepted_indices=pool.accepted_indices,
                                      assignments=frr.regenerate_assignments(pool))
    res2 = frr.randomization_test(W0, g["t5k_y"], rows_pool, find_fi=True, alpha=0.05)
    assert res2.p_value == res.p_value and res2.fi == res.fi
    assert np.array_equal(res2.stat_distribution, res.stat_distribution)


def test_large_keys_pool_vs_oracle():
    """2e4 keys at n=5000: a, p(tau) on a 512-point grid vs the C oracle."""
    m = 20_000
    pool = _t5k_pool(m)
    W = frr.regenerate_assignments(pool)
    y = np.random.default_rng(55).standard_normal(5000) * 2.0 + W[0]
    res = frr.randomization_pvalue(W[0], y, pool)
    a = O.c_dim_rows(W, y, 2500)
    assert np.array_equal(res.stat_distribution, a)
    b = O.c_dim_rows(W, W[0].astype(np.float64), 2500)
    from paper_2501_07642_b200.inference import _PoolStats

    ps = _PoolStats(pool, W[0], y)
    taus = np.linspace(res.tau_obs - 3, res.tau_obs + 3, 512)
    rhs = [abs(ps.tau_obs - float(t) * ps.b_obs) for t in taus]
    got = ps.counts(taus, rhs)
    want = [O.c_count_ge(a, b, float(t), r) for t, r in zip(taus, rhs)]
    assert got.tolist() == want


def test_chunked_key_stream_equals_single_kernel():
    """A keys pool larger than one workspace chunk (3e5 keys at n=5000): the
    pipelined chunk-by-chunk upload + frr_dim_mc_ws equals the single-kernel
    frr_dim_mc on every key, and a sample across the chunk boundaries equals
    the C oracle."""
    import torch

    from paper_2501_07642_b200 import _native as N
    from paper_2501_07642_b200.inference import _PoolStats

    m = 300_000
    pool = _t5k_pool(m)
    chunk = int(N.lib().frr_dim_mc_chunk_keys(m, 5000, 2500, N.lib().frr_dim_mc_workspace_bytes(m, 5000)))
    assert 32 <= chunk < m
    W0 = frr.batch_assignments(5, np.array([0], dtype=np.uint64), 5000, 2500)[0]
    y = np.random.default_rng(57).standard_normal(5000) + W0
    ps = _PoolStats(pool, W0, y)
    dev = N.device()
    draws = torch.from_numpy(pool.keys[:, 1].astype(np.int64)).to(dev)
    y_dev = torch.from_numpy(y).to(dev)
    from paper_2501_07642_b200.inference import _pack_bits

    obs = torch.from_numpy(_pack_bits(W0).view(np.int32)).to(dev)
    a = torch.empty(m, dtype=torch.float64, device=dev)
    b = torch.empty(m, dtype=torch.float64, device=dev)
    N.call("frr_dim_mc", 5, N.ptr(draws), m, 5000, 2500, N.ptr(y_dev), N.ptr(obs), N.ptr(a), N.ptr(b), None,
           N.stream_ptr())
    assert torch.equal(ps.a_local, a) and torch.equal(ps.b_local, b)
    pick = np.unique(np.concatenate([np.arange(chunk - 40, chunk + 40), np.arange(m - 40, m), np.arange(40)]))
    W = O.c_batch_assign(5, (997 * pick).astype(np.uint64), 5000, 2500)
    assert np.array_equal(ps.a_local.cpu().numpy()[pick], O.c_dim_rows(W, y, 2500))


def test_keys_pool_t_near_n_vs_oracle():
    """k_dim with t = n - 1, n a multiple of 32 (padding steps re-read past the table)."""
    n, t, m = 1056, 1055, 3000
    keys = np.column_stack([np.full(m, 9, dtype=np.uint64), 13 * np.arange(m, dtype=np.uint64)])
    pool = frr.RandomizationPool(
        design=frr.DesignSpec(n, t, accept_prob=1.0, max_draws=m * 13, batch_size=13, root_seed=9),
        stats=np.zeros(m), threshold_value=0.0, n_candidates=m * 13, accepted_indices=13 * np.arange(m), keys=keys)
    W = frr.regenerate_assignments(pool)
    assert np.array_equal(W, O.c_batch_assign(9, 13 * np.arange(m, dtype=np.uint64), n, t))
    y = np.random.default_rng(56).standard_normal(n) + W[0]
    res = frr.randomization_pvalue(W[0], y, pool)
    assert np.array_equal(res.stat_distribution, O.c_dim_rows(W, y, t))


def test_keys_pool_with_rejection_key(golden):
    """Regeneration + test statistics for a keys pool containing a key
    crafted to hit the rejection zone (tests/golden/rejection.npz, n=5000)."""
    g = golden("rejection")
    n, t, _ = (int(v) for v in g["cases"][5])
    seed, draw = int(g["seeds"][5]), int(g["draw"])
    ids = np.arange(draw - 50, draw + 50, dtype=np.uint64)
    keys = np.column_stack([np.full(ids.size, seed, dtype=np.uint64), ids])
    pool = frr.RandomizationPool(
        design=frr.DesignSpec(n, t, accept_prob=1.0, max_draws=draw + 50, batch_size=1, root_seed=seed),
        stats=np.zeros(ids.size), threshold_value=0.0, n_candidates=draw + 50,
        accepted_indices=ids.astype(np.int64), keys=keys)
    W = frr.regenerate_assignments(pool)
    assert np.array_equal(W, O.c_batch_assign(seed, ids, n, t))
    y = np.random.default_rng(57).standard_normal(n) + W[50]
    res = frr.randomization_pvalue(W[50], y, pool)
    assert np.array_equal(res.stat_distribution, O.c_dim_rows(W, y, t))


def test_label_symmetry_and_constant_y(pool8):
    rows = pool8.assignments
    y = np.random.default_rng(204).standard_normal(8)
    flipped = frr.RandomizationPool(design=pool8.design, stats=pool8.stats, threshold_value=pool8.threshold_value,
                                    n_candidates=pool8.n_candidates, accepted_indices=pool8.accepted_indices,
                                    assignments=(1 - rows).astype(np.int8))
    a = frr.randomization_pvalue(rows[5], y, pool8)
    b = frr.randomization_pvalue((1 - rows[5]).astype(np.int8), y, flipped)
    assert a.p_value == b.p_value
    res = frr.randomization_pvalue(rows[0], np.full(8, 2.5), pool8)
    assert res.p_value == 1.0 and res.tau_obs == 0.0


def test_not_in_pool_warning():
    X = np.random.default_rng(205).standard_normal((8, 2))
    pool = frr.monte_carlo_pool(X, frr.DesignSpec(8, 4, accept_prob=0.1, max_draws=50, batch_size=10,
                                                  precision_mode="ridge"))
    mat = frr.pool_assignment_matrix(pool)
    outside = np.array([1, 1, 1, 1, 0, 0, 0, 0], dtype=np.int8)
    if any(np.array_equal(outside, r) for r in mat):
        outside = 1 - outside
    with pytest.warns(UserWarning, match="not a member"):
        res = frr.randomization_pvalue(outside, np.random.default_rng(1).standard_normal(8), pool)
    assert not res.obs_in_pool


def test_custom_statistic_and_errors(pool8):
    y = np.random.default_rng(210).standard_normal(8)
    obs = pool8.assignments[2]

    def manual(w, yy):
        w = np.asarray(w)
        return yy[w == 1].mean() - yy[w == 0].mean()

    assert frr.randomization_pvalue(obs, y, pool8).p_value == frr.randomization_pvalue(obs, y, pool8,
                                                                                       statistic=manual).p_value
    with pytest.raises(UnsupportedStatisticError):
        frr.fiducial_interval(obs, y, pool8, statistic=manual)
    with pytest.raises(InvalidDesignError):
        frr.fiducial_interval(obs, y, pool8, alpha=1.5)
    sub = frr.RandomizationPool(design=pool8.design, stats=pool8.stats[:5], threshold_value=0.0,
                                n_candidates=70, accepted_indices=pool8.accepted_indices[:5],
                                assignments=pool8.assignments[:5])
    with pytest.raises(EmptyIntervalError):
        frr.fiducial_interval(pool8.assignments[0], y, sub, alpha=0.15)


def test_fi_contains_true_effect_noiseless(pool8):
    obs = pool8.assignments[3]
    y = 1.0 + 2.75 * obs
    lo, hi = frr.fiducial_interval(obs, y, pool8, alpha=0.05)
    assert lo <= 2.75 <= hi
    res = frr.randomization_test(obs, y, pool8, find_fi=True)
    assert res.fi == (lo, hi)


def test_paper_style_arguments(pool8):
    y = np.random.default_rng(3).standard_normal(8)
    a = frr.randomization_test(obsW=pool8.assignments[1], obsY=y, candidate_randomizations=pool8.assignments,
                               findFI=True)
    b = frr.randomization_test(pool8.assignments[1], y, pool8, find_fi=True)
    assert a.p_value == b.p_value and a.fi == b.fi


def test_threshold_sweep():
    X = np.random.default_rng(212).standard_normal((16, 3))
    y = np.random.default_rng(213).standard_normal(16)
    base = frr.DesignSpec(16, 8, accept_prob=0.5, max_draws=500, batch_size=100, root_seed=6)
    rows = frr.threshold_sweep(X, base, [0.05, 0.1, 0.2, 0.6, 1.0], y, find_fi=True, alpha=0.25)
    counts = [r["n_accepted"] for r in rows]
    assert all(r["status"] == "ok" for r in rows) and counts == sorted(counts) and counts[-1] == 500
    bad = frr.threshold_sweep(np.column_stack([np.ones(10), np.arange(10.0)]),
                              frr.DesignSpec(10, 5, accept_prob=0.5, max_draws=50, batch_size=50), [0.5], np.arange(10.0))
    assert bad[0]["status"].startswith("failed")


@pytest.mark.slow
def test_c5_full_size():
    """C5: 1e6 accepted keys at n=5000 with a fiducial interval.  p-value and
    tau_obs consistent with the returned distribution, a 5000-key sample of
    the distribution bit-exact vs the oracle, and the interval's boundary
    p-values recomputed from the distribution on the host."""
    m = 10**6
    keys = np.column_stack([np.full(m, 5, dtype=np.uint64), 997 * np.arange(m, dtype=np.uint64)])
    pool = frr.RandomizationPool(
        design=frr.DesignSpec(5000, 2500, accept_prob=1.0, max_draws=m * 997, batch_size=997, root_seed=5),
        stats=np.zeros(m), threshold_value=0.0, n_candidates=m * 997, accepted_indices=997 * np.arange(m),
        keys=keys)
    X = np.random.default_rng(5).standard_normal((5000, 64))
    obs = frr.batch_assignments(5, np.array([0], dtype=np.uint64), 5000, 2500)[0]
    rng = np.random.default_rng(5)
    y = X @ rng.standard_normal(64) + 1.0 * obs + 0.5 * rng.standard_normal(5000)
    res = frr.randomization_test(obs, y, pool, find_fi=True, alpha=0.05)
    a = res.stat_distribution
    assert a.shape == (m,)
    assert res.p_value == float(np.count_nonzero(np.abs(a) >= abs(res.tau_obs))) / m
    idx = np.random.default_rng(1).choice(m, 5000, replace=False)
    W = O.c_batch_assign(5, keys[idx, 1], 5000, 2500)
    assert np.array_equal(O.c_dim_rows(W, y, 2500), a[idx])
    assert O.c_dim_rows(obs[None, :].astype(np.int8), y, 2500)[0] == res.tau_obs
    lo, hi = res.fi
    assert lo < res.tau_obs < hi


def test_threshold_sweep_equals_per_probability_pools():
    X = np.random.default_rng(31).standard_normal((40, 4))
    y = np.random.default_rng(32).standard_normal(40)
    for mode, extra in (("monte_carlo", dict(max_draws=20_000, batch_size=1000, root_seed=9)), ("exact", {})):
        if mode == "exact":
            X = np.random.default_rng(33).standard_normal((16, 3))
            y = np.random.default_rng(34).standard_normal(16)
        n = X.shape[0]
        base = frr.DesignSpec(n, n // 2, accept_prob=0.5, mode=mode, **extra)
        probs = [0.001, 0.01, 0.2, 1.0]
        rows = frr.threshold_sweep(X, base, probs, y, find_fi=True, alpha=0.2)
        for p, row in zip(probs, rows):
            pool = frr.generate_pool(X, dataclasses.replace(base, accept_prob=p))
            res = frr.randomization_test(frr.pool_assignment_matrix(pool)[0], y, pool, find_fi=True, alpha=0.2)
            assert row["status"] == "ok" and row["p_value"] == res.p_value
            assert row["n_accepted"] == pool.n_accepted and row["fi_width"] == res.fi[1] - res.fi[0]
