"""The product's multi-rank path with the real kernels: two ranks share the
one B200 of the test box over a gloo group (CUDA tensors staged through the
host by TorchComm; NCCL is the production backend, one GPU per rank).

Every collective of the product path runs: the all-gathered threshold
sample and the all-reduced narrowing counts, the 8 all-reduced radix
histograms, the tie-count all-gather and the rank-ordered gather of the
accepted (index, statistic) pairs (DeviceSelectOps + libfrr kernels), the
agreed fused-exact bound, and for the randomization test the all-reduced
p(tau) counts and the gathered test statistics.  Pools, p-values and
fiducial intervals must equal the world-size-1 results bit for bit -- the
analogue of the reference's invariance test (test_acceptance.py:247-267)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _case(name):
    import paper_2501_07642_b200 as frr

    if name == "c2_prefix":  # C2 shape, enough draws for the sampled narrowing (>= 2^22)
        X = np.random.default_rng(2).standard_normal((1000, 64))
        d = frr.DesignSpec(1000, 500, accept_prob=1e-3, max_draws=5_000_000, batch_size=10_000, root_seed=42)
        p = frr.monte_carlo_pool(X, d)
        return {"idx": p.accepted_indices, "stats": p.stats, "thr": np.array([p.threshold_value]),
                "keys": p.keys}
    if name == "exact_fused":  # split enumeration fused with the narrowing (the C4 path), n=26
        X = np.random.default_rng(26).standard_normal((26, 5))
        d = frr.DesignSpec(26, 13, accept_prob=1e-3, mode="exact")
        p = frr.enumerate_exact(X, d)
        return {"idx": p.accepted_indices, "stats": p.stats, "thr": np.array([p.threshold_value]),
                "rows": p.assignments}
    if name == "c5_keys":  # C5 shape: keys pool, test + fiducial interval
        n, t, m = 5000, 2500, 20_000
        rng = np.random.default_rng(5)
        X = rng.standard_normal((n, 8))
        design = frr.DesignSpec(n, t, accept_prob=1.0, max_draws=m, root_seed=5)
        draws = (np.arange(m, dtype=np.uint64) * np.uint64(997))
        pool = frr.RandomizationPool(design=design, stats=np.zeros(m), threshold_value=0.0, n_candidates=m,
                                     accepted_indices=draws.astype(np.int64),
                                     keys=np.column_stack([np.full(m, 5, dtype=np.uint64), draws]))
        obs = frr.batch_assignments(5, draws[:1], n, t)[0]
        y = X @ rng.standard_normal(8) + 1.0 * obs + 0.5 * rng.standard_normal(n)
        r = frr.randomization_test(obs, y, pool, find_fi=True)
        return {"p": np.array([r.p_value]), "tau": np.array([r.tau_obs]), "fi": np.array(r.fi),
                "dist": r.stat_distribution, "in_pool": np.array([r.obs_in_pool])}
    raise KeyError(name)


CASES = ("c2_prefix", "exact_fused", "c5_keys")


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)  # both ranks on the test box's one GPU
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2501_07642_b200._select import TorchComm, default_comm

        assert isinstance(default_comm(), TorchComm) and default_comm().world == world
        out[rank] = {c: _case(c) for c in CASES}
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def results():
    import torch.multiprocessing as mp

    want = {c: _case(c) for c in CASES}  # world size 1 (no process group here)
    with mp.Manager() as man:
        out = man.dict()
        mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
        got = {r: dict(v) for r, v in dict(out).items()}
    return want, got


@pytest.mark.parametrize("case", CASES)
def test_two_ranks_equal_one(results, case):
    want, got = results
    for rank in (0, 1):
        g, w = got[rank][case], want[case]
        assert set(g) == set(w)
        for k in w:
            if w[k] is None:
                assert g[k] is None, (case, rank, k)
            else:
                assert np.array_equal(np.asarray(g[k]), np.asarray(w[k])), (case, rank, k)
    if case == "c2_prefix":
        assert want[case]["idx"].shape[0] == 5000
