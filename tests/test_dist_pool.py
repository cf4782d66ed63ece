"""Multi-rank pool construction (NCCL on the GPU path) over gloo on CPU:
generation._Pass1's candidate sharding, the global select and the pool
assembly at world sizes 2 and 3 must give exactly the world-size-1 pool, and
_PoolStats' rank-ordered gather of the test statistics must reassemble them
(the counts of p(tau) are all-reduced: tests/test_gpu_multirank.py).
The per-rank GPU compute (pass-1 statistics, select kernels, exact rows) is
replaced by the C oracle / numpy checker ops; the orchestration under test
is the product's."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import paper_2501_07642_b200 as frr
from paper_2501_07642_b200 import generation as G
from paper_2501_07642_b200._select import select_k_smallest
from paper_2501_07642_b200.inference import _PoolStats
from select_ops import NumpySelectOps


def _patch_compute(setattr_=setattr):
    def mc_stats(kernel, design, lo, count, out=None):
        bal = O.Balance(kernel._zq, kernel._inv_scale_sq)
        return torch.from_numpy(O.c_mc_stats(bal, design.n_treated, design.root_seed, lo, count, threads=1))

    def exact_stats(kernel, design, lo, count, out=None):
        bal = O.Balance(kernel._zq, kernel._inv_scale_sq)
        return torch.from_numpy(O.c_exact_stats(bal, design.n_treated, lo, count, threads=1))

    def select(stats, lo, k, comm, keep_device=False, keys_seed=None, m_total=None):
        idx, val, thr = select_k_smallest(stats, lo, k, NumpySelectOps(), comm)
        if keys_seed is not None:
            keys = np.column_stack([np.full(idx.shape[0], keys_seed, dtype=np.uint64), idx.numpy().astype(np.uint64)])
            return idx.numpy(), val.numpy(), thr, keys
        if keep_device:  # the "device" copy of the accepted ranks feeds exact_rows_device
            return idx.numpy(), val.numpy(), thr, idx.numpy().astype(np.uint64)
        return idx.numpy(), val.numpy(), thr

    setattr_(G, "mc_stats_device", mc_stats)
    setattr_(G, "exact_stats_device", exact_stats)
    setattr_(G, "_select_device", select)
    setattr_(G, "exact_rows_device", lambda ranks, n, t: torch.from_numpy(O.c_exact_rows(ranks, n, t)))


CASES = {
    "mc": (np.random.default_rng(21).standard_normal((12, 3)),
           dict(n_units=12, n_treated=6, accept_prob=0.05, max_draws=4001, batch_size=97, root_seed=21)),
    "mc_ties": (np.random.default_rng(3).standard_normal((10, 1)),
                dict(n_units=10, n_treated=5, accept_prob=0.3, max_draws=1000, batch_size=25,
                     precision_mode="diagonal", root_seed=3)),
    "exact": (np.random.default_rng(102).standard_normal((14, 3)),
              dict(n_units=14, n_treated=7, accept_prob=0.03, mode="exact")),
}


def _patch_fused(setattr_, variant):
    """Exact pass 1 fused with the narrowing (generation.exact_narrowed_device)
    on every shard, whatever its size: the sample and filter kernels replaced
    by the oracle, the filter's output shuffled (the kernel appends in no
    particular order).  variant "low": a bound below the threshold, so every
    rank must agree to fall back to the full statistics."""
    from paper_2501_07642_b200 import _select as S

    def shard_stats(kernel, design, lo, count):
        bal = O.Balance(kernel._zq, kernel._inv_scale_sq)
        return O.c_exact_stats(bal, design.n_treated, lo, count, threads=1)

    def sample(kernel, design, lo, stride, s_r):
        return torch.from_numpy(shard_stats(kernel, design, lo, stride * s_r)[::stride].copy())

    def filt(kernel, design, lo, count, h, cap):
        st = shard_stats(kernel, design, lo, count)
        keep = np.flatnonzero(st.view(np.uint64) <= np.uint64(h))
        keep = np.random.default_rng(lo).permutation(keep)
        idx, val = lo + keep[:cap], st[keep[:cap]]
        return torch.from_numpy(idx.astype(np.int64)), torch.from_numpy(val.copy()), int(keep.size)

    def sort_by_rank(ranks, vals, rank_end):  # checker stand-in for frr_sort_pairs
        order = np.argsort(ranks.numpy(), kind="stable")
        return ranks[order].contiguous(), vals[order].contiguous()

    setattr_(G, "_sort_by_rank", sort_by_rank)
    setattr_(G, "_use_fused_select", lambda design, d, m, k: design.mode == "exact")
    setattr_(G, "_narrow_sample", sample)
    setattr_(G, "_narrow_filter", filt)
    setattr_(G, "_select_ops", NumpySelectOps)
    setattr_(S, "SAMPLE", 600)
    if variant == "low":
        setattr_(S, "bound_from_sample", lambda *a: (0, 0.0))


def _build(name):
    X, kw = CASES[name.split(":")[0]]
    design = frr.DesignSpec(**kw)
    pool = frr.generate_pool(X, design)
    return (pool.accepted_indices, pool.stats, pool.threshold_value,
            None if pool.assignments is None else pool.assignments, None if pool.keys is None else pool.keys)


def _worker(rank, world, port, name, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _patch_compute()
        if ":" in name:
            _patch_fused(setattr, name.split(":")[1])
        out[rank] = _build(name)
    finally:
        dist.destroy_process_group()


def _gather_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2501_07642_b200._select import TorchComm

        m = 1001
        a = np.arange(m, dtype=np.float64) * 0.5
        lo, hi = m * rank // world, m * (rank + 1) // world
        ga = _PoolStats._gather(TorchComm(), torch.from_numpy(a[lo:hi].copy()))
        out[rank] = ga.numpy()
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("name,world", [("mc", 2), ("mc_ties", 3), ("exact", 2), ("exact:fused", 2),
                                        ("exact:fused", 3), ("exact:low", 2)])
def test_sharded_pool_equals_single_rank(name, world, monkeypatch):
    _patch_compute(monkeypatch.setattr)  # restored after the test
    want = _build(name.split(":")[0])  # world size 1, unfused (no process group in this process)
    with mp.Manager() as man:
        out = man.dict()
        mp.spawn(_worker, args=(world, _free_port(), name, out), nprocs=world, join=True)
        results = dict(out)
    for r in range(world):
        got = results[r]
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1]) and got[2] == want[2]
        for g, w in zip(got[3:], want[3:]):
            assert (g is None and w is None) or np.array_equal(g, w)


def test_pool_stats_gather_rank_order():
    world = 3
    with mp.Manager() as man:
        out = man.dict()
        mp.spawn(_gather_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        results = dict(out)
    for r in range(world):
        assert np.array_equal(results[r], np.arange(1001) * 0.5)


def test_fused_exact_single_rank_equals_unfused(monkeypatch):
    _patch_compute(monkeypatch.setattr)
    want = _build("exact")
    _patch_fused(monkeypatch.setattr, "fused")
    monkeypatch.setattr(G, "exact_stats_device", None)  # the fused path must not need the full array
    got = _build("exact:fused")
    assert all(np.array_equal(g, w) for g, w in zip(got[:2], want[:2])) and got[2] == want[2]
    assert np.array_equal(got[3], want[3])
