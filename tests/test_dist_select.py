"""Multi-rank acceptance selection (NCCL on the GPU path) -- the host
orchestration of _select.select_k_smallest run with world_size 2 over gloo
on CPU.  The per-rank select steps are numpy restatements of the libfrr
kernels (test-side checker ops); the orchestration under test is the
product's: histogram all-reduce per radix pass, tie quota split in rank
order, rank-ordered gather."""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2501_07642_b200 import _select as S
from paper_2501_07642_b200._select import TorchComm, select_k_smallest
from select_ops import NumpySelectOps


def _worker(rank, world, port, stats, p, out, narrow="off"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    if narrow != "off":  # exercise the sampled narrowing (and its fall back) at test sizes
        S.PREFILTER_MIN, S.SAMPLE, S.PREFILTER_MAX_Q = 1, 512, 1.0
        if narrow == "bad-bound":  # h = +0.0: fewer than k statistics under the bound
            def low(sample, k, m_total, ops):
                st = ops.init(1, sample.device)
                ops.set_threshold(st, 0)
                return st, 0.0

            S._bound_state = low
        if narrow == "overflow":  # the true bound with a zero fraction: the capped buffer overflows
            true_state = S._bound_state
            S._bound_state = lambda *a: (true_state(*a)[0], 0.0)
    try:
        M = stats.shape[0]
        lo, hi = M * rank // world, M * (rank + 1) // world
        k = max(1, math.floor(p * M))
        idx, val, thr = select_k_smallest(torch.from_numpy(stats[lo:hi].copy()), lo, k, NumpySelectOps(),
                                          TorchComm())
        out[rank] = (idx.numpy(), val.numpy(), thr)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,ties,p,narrow", [(2, True, 0.1, "off"), (2, False, 0.01, "off"), (3, True, 0.37, "off"),
                                                 (2, False, 0.01, "on"), (3, True, 0.05, "on"),
                                                 (2, True, 0.02, "bad-bound"), (3, False, 0.05, "overflow")])
def test_distributed_select_matches_stable_sort(world, ties, p, narrow):
    rng = np.random.default_rng(world * 7 + ties)
    M = 20011
    stats = np.round(rng.random(M) * (3 if ties else 1e6)) / 7.0
    with mp.Manager() as man:
        out = man.dict()
        mp.spawn(_worker, args=(world, _free_port(), stats, p, out, narrow), nprocs=world, join=True)
        results = dict(out)
    k = max(1, math.floor(p * M))
    order = np.argsort(stats, kind="stable")
    want = np.sort(order[:k])
    for r in range(world):
        idx, val, thr = results[r]
        assert np.array_equal(idx, want)
        assert np.array_equal(val, stats[want])
        assert thr == stats[order[k - 1]]
