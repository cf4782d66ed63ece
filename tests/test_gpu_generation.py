"""GPU pool construction vs the reference's golden pools and the C oracle:
accepted sets, statistics and thresholds bit-exact; size-independent
properties at the full C2 size."""

import dataclasses
import math

import numpy as np
import pytest

import oracle as O
import paper_2501_07642_b200 as frr
from paper_2501_07642_b200 import generation as G
from paper_2501_07642_b200.errors import EnumerationTooLargeError, InvalidDesignError, StorageCapError

pytestmark = pytest.mark.gpu


def test_exact_pool_golden(golden):
    g = golden("pools")
    X = np.random.default_rng(102).standard_normal((10, 3))
    pool = frr.enumerate_exact(X, frr.DesignSpec(10, 5, accept_prob=0.2, mode="exact"))
    assert pool.n_candidates == 252 and pool.n_accepted == 50
    assert np.array_equal(pool.accepted_indices, g["e10_acc"])
    assert np.array_equal(pool.stats, g["e10_stats"]) and pool.threshold_value == float(g["e10_thr"])
    assert np.array_equal(pool.assignments, g["e10_rows"])


def test_c1_golden(golden):
    g = golden("pools")
    X = np.random.default_rng(1).standard_normal((20, 5))
    pool = frr.generate_pool(X, frr.DesignSpec(20, 10, accept_prob=0.01, mode="exact", batch_size=10_000))
    assert pool.n_candidates == 184_756 and pool.n_accepted == 1847
    assert np.array_equal(pool.accepted_indices, g["c1_acc"]) and np.array_equal(pool.stats, g["c1_stats"])
    assert pool.threshold_value == 0.7578915572820588


MC = {
    "mc12a": (100, (12, 3), dict(n_units=12, n_treated=6, accept_prob=0.05, max_draws=2000, batch_size=97, root_seed=21)),
    "mc12all": (100, (12, 3), dict(n_units=12, n_treated=6, accept_prob=1.0, max_draws=2000, batch_size=2000, root_seed=21)),
    "mc12one": (100, (12, 3), dict(n_units=12, n_treated=6, accept_prob=0.01, max_draws=100, batch_size=10, root_seed=9)),
    "mctie": (None, (10, 1), dict(n_units=10, n_treated=5, accept_prob=0.02, max_draws=100, batch_size=25,
                                  precision_mode="diagonal", root_seed=3)),
    "mc20": (105, (20, 5), dict(n_units=20, n_treated=10, accept_prob=0.01, max_draws=100_000, batch_size=20_000,
                                root_seed=12345)),
    "mcridge": (108, (30, 40), dict(n_units=30, n_treated=15, accept_prob=0.1, max_draws=2000, batch_size=500,
                                    precision_mode="ridge", root_seed=31)),
    "mc1000": (2, (1000, 64), dict(n_units=1000, n_treated=500, accept_prob=1e-3, max_draws=20_000,
                                   batch_size=10_000, root_seed=42)),
}


@pytest.mark.parametrize("name", list(MC))
def test_mc_pools_golden(golden, name):
    g = golden("pools")
    xs, shape, kw = MC[name]
    X = np.ones(shape) if xs is None else np.random.default_rng(xs).standard_normal(shape)
    pool = frr.monte_carlo_pool(X, frr.DesignSpec(**kw))
    assert np.array_equal(pool.accepted_indices, g[f"{name}_acc"])
    assert np.array_equal(pool.stats, g[f"{name}_stats"]) and pool.threshold_value == float(g[f"{name}_thr"])
    assert np.array_equal(pool.keys[:, 1], pool.accepted_indices.astype(np.uint64))


def test_tie_break_by_draw_order():
    pool = frr.monte_carlo_pool(np.ones((10, 1)), frr.DesignSpec(10, 5, accept_prob=0.02, max_draws=100,
                                                                 batch_size=25, precision_mode="diagonal", root_seed=3))
    assert pool.accepted_indices.tolist() == [0, 1] and pool.stats[0] == pool.stats[1]


def test_batch_size_and_storage_invariance():
    X = np.random.default_rng(100).standard_normal((12, 3))
    base = frr.DesignSpec(12, 6, accept_prob=0.05, max_draws=2000, batch_size=2000, root_seed=21)
    pools = [frr.monte_carlo_pool(X, dataclasses.replace(base, batch_size=b)) for b in (1, 7, 97, 2000)]
    assert all(G.pools_equal(pools[0], p) for p in pools[1:])
    full = frr.monte_carlo_pool(X, dataclasses.replace(base, storage="full"))
    both = frr.monte_carlo_pool(X, dataclasses.replace(base, storage="both"))
    regen = frr.regenerate_assignments(pools[0])
    assert np.array_equal(regen, full.assignments) and np.array_equal(regen, both.assignments)
    assert full.keys is None and both.keys is not None
    prec = frr.precompute_precision(X, "exact")
    assert np.array_equal(frr.batch_balance(X, prec, regen), pools[0].stats)
    with pytest.raises(InvalidDesignError):
        frr.regenerate_assignments(full)


def test_acceptance_count_law():
    X = np.random.default_rng(100).standard_normal((12, 3))
    rng = np.random.default_rng(103)
    for _ in range(10):
        m = int(rng.integers(1, 2000))
        p = float(rng.uniform(0.0005, 1.0))
        pool = frr.monte_carlo_pool(X, frr.DesignSpec(12, 6, accept_prob=p, max_draws=m, batch_size=min(500, m),
                                                      root_seed=int(rng.integers(0, 2**32))))
        assert pool.n_accepted == max(1, math.floor(p * m))


@pytest.mark.parametrize("M,p,ties", [(1, 1.0, False), (7, 1.0, True), (1000, 0.001, True), (100_003, 0.2, True),
                                      (3_000_017, 1e-3, False), (2_000_000, 0.5, True),
                                      # sampled narrowing (M >= 2^22): distinct values, heavy ties, q at the cut-off
                                      (5_000_011, 1e-3, False), (6_000_000, 1e-4, True), (4_194_304, 0.05, True)])
def test_select_vs_oracle(M, p, ties):
    rng = np.random.default_rng(M)
    st = np.round(rng.random(M) * (5 if ties else 1e12)) / 3.0
    st[: M // 10] = 0.0  # zeros (+0.0) sort first
    acc, thr = G._select(st, p)
    want, wthr = O.c_select(st, p)
    assert np.array_equal(acc, want) and thr == wthr


def test_narrowing_fallback_when_bound_is_low(monkeypatch):
    from paper_2501_07642_b200 import _select as S

    def low(sample, k, m_total, ops):  # h = +0.0: far too low
        st = ops.init(1, sample.device)
        ops.set_threshold(st, 0)
        return st, 0.0

    monkeypatch.setattr(S, "_bound_state", low)
    rng = np.random.default_rng(5)
    st = rng.random(5_000_000) + 0.5
    acc, thr = G._select(st, 1e-3)
    want, wthr = O.c_select(st, 1e-3)
    assert np.array_equal(acc, want) and thr == wthr


def test_narrowing_fallback_when_buffer_overflows(monkeypatch):
    """The true bound with a zero sampled fraction: the capped narrowing
    buffer (4096 entries) overflows, detected at the end of the select."""
    from paper_2501_07642_b200 import _select as S

    true_state = S._bound_state
    monkeypatch.setattr(S, "_bound_state", lambda *a: (true_state(*a)[0], 0.0))
    rng = np.random.default_rng(6)
    st = rng.random(5_000_000)
    acc, thr = G._select(st, 1e-2)
    want, wthr = O.c_select(st, 1e-2)
    assert np.array_equal(acc, want) and thr == wthr


def test_narrowed_select_has_no_host_sync_before_the_end(monkeypatch):
    """The narrowed select reads nothing back until every kernel is queued
    (host stalls during the select then cost no GPU time)."""
    import torch

    from paper_2501_07642_b200 import _select as S
    from paper_2501_07642_b200._select import DeviceSelectOps, LocalComm

    rng = np.random.default_rng(7)
    stats = torch.from_numpy(rng.random(8_000_000)).cuda()
    S.TRACE = []
    try:
        S.select_k_smallest(stats, 0, 8000, DeviceSelectOps(), LocalComm())
        labels = [lab for lab, _ in S.TRACE]
    finally:
        S.TRACE = None
    assert "bound read" not in labels and "compact read" not in labels
    assert labels.index("final launched") < labels.index("narrowed ok")


def test_capped_compaction_reports_full_count():
    """frr_select_compact_capped as the narrowing filter {stat <= h}: only the
    first `cap` entries (index order) are written, n_out is the full count."""
    import torch

    from paper_2501_07642_b200._select import DeviceSelectOps

    rng = np.random.default_rng(8)
    st_h = np.round(rng.random(100_000) * 1000) / 7.0
    stats = torch.from_numpy(st_h).cuda()
    ops = DeviceSelectOps()
    h = float(np.sort(st_h)[5000])
    sth = ops.init(1, stats.device)
    ops.set_threshold(sth, int(np.array([h]).view(np.uint64)[0]))
    everything = torch.full((1,), (1 << 63) - 1, dtype=torch.int64, device=stats.device)
    want = np.flatnonzero(st_h <= h)
    idx, val, n = ops.compact(stats, 17, sth, everything, cap=1000)
    assert int(n.item()) == want.shape[0] and idx.shape[0] == 1000
    assert np.array_equal(idx.cpu().numpy(), want[:1000] + 17) and np.array_equal(val.cpu().numpy(), st_h[want[:1000]])


def test_diagnostic_microbenchmarks_run():
    import ctypes

    import torch

    from paper_2501_07642_b200 import _native as N

    sink = torch.zeros(1, dtype=torch.int64, device="cuda")
    tot, ops = ctypes.c_int64(0), ctypes.c_int64(0)
    N.call("frr_microbench_draws", 64, N.ptr(sink), ctypes.byref(tot), N.stream_ptr())
    N.call("frr_microbench_mma_i8", 192, 1, 16, ctypes.byref(ops), N.stream_ptr())
    torch.cuda.synchronize()
    per_sm = 16 * 4 * 2 * 128 * 192 * 32  # iters x 4 MMAs x 2*M*N*K, one CTA per SM
    assert tot.value > 0 and ops.value > 0 and ops.value % per_sm == 0
    with pytest.raises(InvalidDesignError):
        N.call("frr_microbench_draws", 3, N.ptr(sink), ctypes.byref(tot), N.stream_ptr())


def test_c2_prefix_pool_vs_oracle():
    X = np.random.default_rng(2).standard_normal((1000, 64))
    design = frr.DesignSpec(1000, 500, accept_prob=1e-3, max_draws=200_000, batch_size=10_000, root_seed=42)
    pool = frr.monte_carlo_pool(X, design)
    bal = O.balance_setup(X, O.precision(X, "exact"))
    st = O.c_mc_stats(bal, 500, 42, 0, 200_000)
    acc, thr = O.c_select(st, 1e-3)
    assert np.array_equal(pool.accepted_indices, acc) and np.array_equal(pool.stats, st[acc])
    assert pool.threshold_value == thr


@pytest.mark.slow
def test_c2_full_size_properties():
    """Full C2 (1e8 candidates): accepted count, every accepted statistic
    recomputed by the oracle bit-exactly, and 2e5 random candidates'
    acceptance status consistent with the threshold."""
    X = np.random.default_rng(2).standard_normal((1000, 64))
    design = frr.DesignSpec(1000, 500, accept_prob=1e-3, max_draws=10**8, batch_size=10_000, root_seed=42)
    pool = frr.monte_carlo_pool(X, design)
    assert pool.n_accepted == 100_000
    assert np.all(np.diff(pool.accepted_indices) > 0)
    bal = O.balance_setup(X, O.precision(X, "exact"))
    sample = pool.accepted_indices[:: 10]
    rows = O.c_batch_assign(42, sample.astype(np.uint64), 1000, 500)
    assert np.array_equal(O.c_stats_rows(bal, rows, 500), pool.stats[:: 10])
    assert pool.stats.max() == pool.threshold_value
    rng = np.random.default_rng(9)
    idx = np.unique(rng.integers(0, 10**8, size=200_000))
    rows = O.c_batch_assign(42, idx.astype(np.uint64), 1000, 500)
    st = O.c_stats_rows(bal, rows, 500)
    accepted = np.isin(idx, pool.accepted_indices)
    assert np.all(accepted[st < pool.threshold_value])
    assert not np.any(accepted[st > pool.threshold_value])


def test_exact_cap_and_storage_cap():
    X = np.random.default_rng(106).standard_normal((20, 2))
    with pytest.raises(EnumerationTooLargeError):
        frr.enumerate_exact(X, frr.DesignSpec(20, 10, accept_prob=0.1, mode="exact", enumeration_cap=1000))
    X12 = np.random.default_rng(100).standard_normal((12, 3))
    with pytest.raises(StorageCapError):
        frr.monte_carlo_pool(X12, frr.DesignSpec(12, 6, accept_prob=0.5, max_draws=1000, batch_size=100,
                                                 storage="full", full_storage_cap=100))


def test_pool_files_streaming_and_round_trip(tmp_path):
    X = np.random.default_rng(100).standard_normal((12, 3))
    base = frr.DesignSpec(12, 6, accept_prob=0.2, max_draws=300, batch_size=32, root_seed=19, storage="full")
    streamed = tmp_path / "s.csv"
    pool = frr.monte_carlo_pool(X, base, out_path=streamed)
    assert pool.assignments is None
    held = frr.monte_carlo_pool(X, base)
    written = tmp_path / "h.csv"
    frr.write_pool(held, written)
    assert streamed.read_bytes() == written.read_bytes()
    for storage in ("keys", "both"):
        d = dataclasses.replace(base, storage=storage)
        p = frr.monte_carlo_pool(X, d)
        path = tmp_path / f"{storage}.csv"
        frr.write_pool(p, path)
        back = frr.read_pool(path)
        assert np.array_equal(frr.pool_assignment_matrix(back), frr.pool_assignment_matrix(p))
    Xe = np.random.default_rng(107).standard_normal((9, 2))
    de = frr.DesignSpec(9, 4, accept_prob=0.3, mode="exact", batch_size=17)
    a, b = tmp_path / "ea.csv", tmp_path / "eb.csv"
    frr.enumerate_exact(Xe, de, out_path=a)
    frr.write_pool(frr.enumerate_exact(Xe, de), b)
    assert a.read_bytes() == b.read_bytes()


def test_paper_api_generate_randomizations(tmp_path):
    X = np.random.default_rng(3).standard_normal((20, 3))
    r = frr.generate_randomizations(n_units=20, n_treated=10, X=X, randomization_accept_prob=0.01,
                                    max_draws=10_000, batch_size=1000, randomization_type="monte_carlo", seed=5)
    assert r.randomizations.shape == (100, 20) and np.array_equal(r.balance, r.stats)
    e = frr.generate_randomizations(10, 5, np.random.default_rng(4).standard_normal((10, 3)),
                                    randomization_type="exact", randomization_accept_prob=0.2)
    assert e.randomizations.shape == (50, 10)
    hi = frr.generate_randomizations(30, 15, np.random.default_rng(5).standard_normal((30, 40)),
                                     max_draws=500, batch_size=500, approximate_inv=True)
    assert hi.design.precision_mode == "ridge"


@pytest.mark.slow
def test_c4_full_size_properties():
    """C4 (exact n=34, t=17: 2,333,606,220 ranks, d=5, p=1e-3) on one GPU:
    accepted count, every 50th accepted statistic and 200 random windows
    of 500 consecutive ranks recomputed by the oracle bit-exactly, and the
    windows' acceptance status consistent with the threshold."""
    X = np.random.default_rng(4).standard_normal((34, 5))
    design = frr.DesignSpec(34, 17, accept_prob=1e-3, mode="exact", enumeration_cap=3 * 10**9)
    pool = frr.enumerate_exact(X, design)
    total = math.comb(34, 17)
    assert pool.n_candidates == total == 2_333_606_220
    assert pool.n_accepted == math.floor(1e-3 * total)
    assert np.all(np.diff(pool.accepted_indices) > 0)
    assert np.all(pool.assignments.sum(axis=1) == 17)
    bal = O.balance_setup(X, O.precision(X, "exact"))
    sub = pool.accepted_indices[::50]
    rows = O.c_exact_rows(sub.astype(np.uint64), 34, 17)
    assert np.array_equal(rows, pool.assignments[::50])
    assert np.array_equal(O.c_stats_rows(bal, rows, 17), pool.stats[::50])
    rng = np.random.default_rng(11)
    acc = set(pool.accepted_indices.tolist())
    for lo in rng.integers(0, total - 500, size=200):
        st = O.c_exact_stats(bal, 17, int(lo), 500)
        for i, s in enumerate(st):
            if s < pool.threshold_value:
                assert int(lo) + i in acc
            elif s > pool.threshold_value:
                assert int(lo) + i not in acc


def test_c3_sampled_parity_around_threshold():
    """C3 shape (n=2000, d=1024, ridge; the N-tiled tensor-core kernel) on a
    3e5-draw prefix: the pool equals the oracle's selection over GPU stats
    that are bit-exact on every accepted draw, the 1000 ranks either side of
    the threshold and 1000 random draws (SURVEY 8(d) sampled parity)."""
    X = np.random.default_rng(3).standard_normal((2000, 1024))
    M, p = 300_000, 1e-4
    design = frr.DesignSpec(2000, 1000, accept_prob=p, max_draws=M, batch_size=10_000, root_seed=43,
                            precision_mode="ridge")
    pool = frr.monte_carlo_pool(X, design)
    kern = frr.precompute_precision(X, "ridge")._kernel
    assert kern.tc_plan()[0] == 2  # N-tiled kernel serves this shape
    st = G.mc_stats_device(kern, design, 0, M).cpu().numpy()
    k = G._accepted_count(p, M)
    order = np.argsort(st, kind="stable")
    acc = np.sort(order[:k])
    assert np.array_equal(pool.accepted_indices, acc) and np.array_equal(pool.stats, st[acc])
    assert pool.threshold_value == st[order[k - 1]]
    rng = np.random.default_rng(33)
    idx = np.unique(np.concatenate([order[: k + 1000], rng.integers(0, M, size=1000)]))
    bal = O.balance_setup(X, O.precision(X, "ridge"))
    rows = O.c_batch_assign(43, idx.astype(np.uint64), 2000, 1000)
    want = O.c_stats_rows(bal, rows, 1000)
    assert np.array_equal(st[idx].view(np.uint64), want.view(np.uint64))


def _exact_pool_both(X, design, monkeypatch):
    fused = frr.enumerate_exact(X, design)
    monkeypatch.setenv("FRR_EXACT_FUSED_SELECT", "0")
    plain = frr.enumerate_exact(X, design)
    monkeypatch.delenv("FRR_EXACT_FUSED_SELECT")
    return fused, plain


@pytest.mark.parametrize("integer_x", [False, True])
def test_fused_exact_select_vs_oracle(monkeypatch, integer_x):
    """Exact pass 1 fused with the narrowing (frr_exact_stats_split_filtered)
    against the oracle's full statistics + stable-argsort select, n=24
    (2,704,156 ranks); integer X makes many statistics tie at the threshold."""
    from paper_2501_07642_b200 import _select as S
    monkeypatch.setattr(S, "PREFILTER_MIN", 1 << 20)
    rng = np.random.default_rng(24)
    X = rng.integers(-2, 3, size=(24, 5)).astype(np.float64) if integer_x else rng.standard_normal((24, 5))
    design = frr.DesignSpec(24, 12, accept_prob=2e-3, mode="exact")
    fused, plain = _exact_pool_both(X, design, monkeypatch)
    assert G.pools_equal(fused, plain) and np.array_equal(fused.assignments, plain.assignments)
    bal = O.balance_setup(X, O.precision(X, "exact"))
    st = O.c_exact_stats(bal, 12, 0, math.comb(24, 12))
    want, wthr = O.c_select(st, 2e-3)
    assert np.array_equal(fused.accepted_indices, want) and fused.threshold_value == wthr
    assert np.array_equal(fused.stats, st[want])


@pytest.mark.parametrize("bound", ["low", "overflow"])
def test_fused_exact_select_fallbacks(monkeypatch, bound):
    """A bound below the threshold (fewer than k kept) falls back to the full
    statistics array; a kept buffer that overflows (here: sized for 1000
    pairs) is refilled with the exact count, without the fallback."""
    from paper_2501_07642_b200 import _select as S
    monkeypatch.setattr(S, "PREFILTER_MIN", 1 << 20)
    h = 0 if bound == "low" else 0x7FF0000000000000  # +0.0 / +inf
    monkeypatch.setattr(S, "bound_from_sample", lambda *a: (h, 0.0))
    calls, caps = [], []
    real = G.exact_stats_device
    monkeypatch.setattr(G, "exact_stats_device", lambda *a, **kw: calls.append(1) or real(*a, **kw))
    real_filter = G._narrow_filter

    def record(kernel, design, lo, count, hb, cap):
        caps.append(cap)
        return real_filter(kernel, design, lo, count, hb, cap)

    monkeypatch.setattr(G, "_narrow_filter", record)
    monkeypatch.setattr(G, "KEPT_SLACK", 0.0)  # first buffer: 1000 pairs
    monkeypatch.setattr(G, "KEPT_PAD", 1000)
    X = np.random.default_rng(3).standard_normal((26, 5))
    design = frr.DesignSpec(26, 13, accept_prob=1e-3, mode="exact")
    fused = frr.enumerate_exact(X, design)
    if bound == "low":
        assert calls == [1]  # the fallback ran pass 1 unfused
    else:
        assert calls == [] and caps == [1000, math.comb(26, 13)], caps  # rerun with the exact count
    monkeypatch.undo()
    monkeypatch.setenv("FRR_EXACT_FUSED_SELECT", "0")
    plain = frr.enumerate_exact(X, design)
    assert G.pools_equal(fused, plain)


def test_fused_exact_select_n26_matches_unfused(monkeypatch):
    """n=26, t=13 (10,400,600 ranks): above PREFILTER_MIN with the default
    constants, so enumerate_exact takes the fused path as C4 does."""
    X = np.random.default_rng(26).standard_normal((26, 5))
    design = frr.DesignSpec(26, 13, accept_prob=1e-3, mode="exact")
    fused, plain = _exact_pool_both(X, design, monkeypatch)
    assert fused.n_accepted == math.floor(1e-3 * math.comb(26, 13))
    assert G.pools_equal(fused, plain) and np.array_equal(fused.assignments, plain.assignments)


@pytest.mark.parametrize("n,t,lo,stride", [(34, 17, 0, 2225), (34, 17, 123_456_789, 999_983), (26, 13, 5, 1),
                                           (27, 9, 17, 4099)])
def test_split_strided_sample_vs_oracle(n, t, lo, stride):
    """The fused path's sample kernel: statistics of ranks lo + j * stride."""
    import paper_2501_07642_b200._native as NAT
    X = np.random.default_rng(n + t).standard_normal((n, 5))
    design = frr.DesignSpec(n, t, accept_prob=1e-3, mode="exact", enumeration_cap=3 * 10**9)
    kern = frr.precompute_precision(X, "exact")._kernel
    m = min(4096, (math.comb(n, t) - lo + stride - 1) // stride)
    got = G._narrow_sample(kern, design, lo, stride, m).cpu().numpy()
    bal = O.balance_setup(X, O.precision(X, "exact"))
    ranks = lo + stride * np.arange(m, dtype=np.uint64)
    rows = O.c_exact_rows(ranks.astype(np.uint64), n, t)
    assert np.array_equal(got, O.c_stats_rows(bal, rows, t))
    assert NAT.lib().frr_exact_stats_split_strided  # exported


@pytest.mark.parametrize("shape,dtype", [((2333606, 34), "int8"), ((2333606,), "int64"), (((1 << 18) + 3,), "float64"),
                                         ((77, 3), "int8"), ((40_000_001,), "float64")])
def test_staged_to_host_pipelined(shape, dtype):
    """_native.to_host (chunked DMA through the page-locked stage, host copies
    overlapped) returns exactly the tensor's contents."""
    import torch
    import paper_2501_07642_b200._native as NAT
    g = torch.Generator(device="cuda").manual_seed(7)
    t = torch.randint(-100, 100, shape, dtype=getattr(torch, dtype), device="cuda", generator=g)
    if dtype == "float64":
        t = t * 0.37
    for _ in range(2):
        got = NAT.to_host(t)
        assert got.dtype == t.cpu().numpy().dtype and np.array_equal(got, t.cpu().numpy())


@pytest.mark.parametrize("n,t,d,lo,hi", [(24, 12, 5, 0, None), (27, 9, 3, 12_345, 3_000_001), (26, 13, 8, 777, None),
                                         (30, 15, 16, 10**8, 10**8 + 2_000_003)])
def test_tiled_filter_equals_rank_order_filter(monkeypatch, n, t, d, lo, hi):
    """frr_exact_tiled_filtered keeps exactly the (rank, stat) pairs of
    frr_exact_stats_split_filtered on a shard [lo, hi) that cuts blocks,
    widths 4/6/8/16; n=24 also against the oracle's statistics."""
    X = np.random.default_rng(n * d).standard_normal((n, d))
    design = frr.DesignSpec(n, t, accept_prob=1e-3, mode="exact", enumeration_cap=3 * 10**9)
    kern = frr.precompute_precision(X, "exact")._kernel
    hi = math.comb(n, t) if hi is None else hi
    count = hi - lo
    samp = G._narrow_sample(kern, design, lo, max(1, count // 4096), 4096).cpu().numpy()
    h = int(np.quantile(samp, 0.01, method="lower").view(np.uint64)) if samp.size else 0
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("FRR_EXACT_TILED", mode)
        idx, val, nk = G._narrow_filter(kern, design, lo, count, h, count // 20 + 4096)
        o = np.argsort(idx[:nk].cpu().numpy())
        out[mode] = (idx[:nk].cpu().numpy()[o], val[:nk].cpu().numpy()[o], nk)
    assert out["1"][2] == out["0"][2] > 0
    assert np.array_equal(out["1"][0], out["0"][0]) and np.array_equal(out["1"][1], out["0"][1])
    if n == 24:
        bal = O.balance_setup(X, O.precision(X, "exact"))
        st = O.c_exact_stats(bal, t, 0, count)
        want = np.flatnonzero(st.view(np.uint64) <= np.uint64(h))
        assert np.array_equal(out["1"][0], want) and np.array_equal(out["1"][1], st[want])


def test_c4_fused_pool_equals_unfused_full_size(monkeypatch):
    """C4 at full size (2,333,606,220 ranks): the fused tiled path's pool is
    the unfused path's (18.7 GB statistics array + select), which the
    full-size parity run checked against the oracle (profiles/r01f_full_parity_c4.json)."""
    X = np.random.default_rng(4).standard_normal((34, 5))
    design = frr.DesignSpec(34, 17, accept_prob=1e-3, mode="exact", enumeration_cap=3 * 10**9)
    fused, plain = _exact_pool_both(X, design, monkeypatch)
    assert fused.n_accepted == 2_333_606
    assert G.pools_equal(fused, plain) and np.array_equal(fused.assignments, plain.assignments)


@pytest.mark.parametrize("n,bits,dups", [(1, 8, False), (2, 1, False), (1000, 8, False), (5000, 20, False),
                                         (3_000_001, 32, False), (100_000, 40, True), (70_000, 64, True)])
def test_sort_pairs_vs_stable_argsort(n, bits, dups):
    """frr_sort_pairs (the fused exact pass's rank ordering) against numpy's
    stable argsort, odd and even pass counts, duplicate keys keep their
    input order."""
    import torch

    from paper_2501_07642_b200 import _native as N

    rng = np.random.default_rng(n + bits)
    hi = (1 << bits) - 1
    if dups:
        keys = rng.integers(0, min(hi, 1000), size=n, dtype=np.uint64, endpoint=True)
    else:  # distinct keys (like ranks), shuffled
        keys = rng.permutation(np.unique(rng.integers(0, hi, size=n, dtype=np.uint64, endpoint=True)))
        n = keys.shape[0]
    vals = np.arange(n, dtype=np.int64)
    k_dev = torch.from_numpy(keys.view(np.int64).copy()).cuda()
    v_dev = torch.from_numpy(vals.copy()).cuda()
    ws_bytes = int(N.lib().frr_sort_pairs_workspace_bytes(n))
    ws = torch.empty(max(1, ws_bytes), dtype=torch.uint8, device="cuda")
    N.call("frr_sort_pairs", N.ptr(k_dev), N.ptr(v_dev), n, bits, N.ptr(ws), ws_bytes, N.stream_ptr())
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(k_dev.cpu().numpy().view(np.uint64), keys[order])
    assert np.array_equal(v_dev.cpu().numpy(), vals[order])


def test_select_start_does_not_wait_for_queued_work():
    """select_start only enqueues: behind a ~100 ms pass 1 it returns in
    milliseconds (a blocking host->device store once made it wait for the
    whole queue), and finish() returns the same selection as the blocking
    select."""
    import time

    import torch

    from paper_2501_07642_b200._select import DeviceSelectOps, LocalComm, select_k_smallest, select_start

    X = np.random.default_rng(2).standard_normal((1000, 64))
    design = frr.DesignSpec(1000, 500, accept_prob=1e-3, max_draws=10**8, batch_size=10_000, root_seed=42)
    kern = frr.precompute_precision(X, "exact")._kernel
    busy = torch.empty(10**8, dtype=torch.float64, device="cuda")
    stats = torch.from_numpy(np.random.default_rng(9).random(8_000_000)).cuda()
    ops, comm = DeviceSelectOps(), LocalComm()
    want = select_k_smallest(stats, 0, 8000, ops, comm)  # also loads every kernel once
    best = float("inf")
    for _ in range(3):  # a host-side hiccup of the VM may hit one attempt; a block hits all
        G.mc_stats_device(kern, design, 0, 10**8, out=busy)
        t0 = time.perf_counter()
        job = select_start(stats, 0, 8000, ops, comm, m_total=stats.shape[0])
        best = min(best, time.perf_counter() - t0)
        got = job.finish()
        assert torch.equal(got[0], want[0]) and torch.equal(got[1], want[1]) and got[2] == want[2]
        if best < 0.03:
            break
    assert best < 0.03, f"select_start blocked for {best * 1e3:.1f} ms"
