"""GPU assignment generation vs the reference's golden keys and the C oracle
(bit-exact)."""

import numpy as np
import pytest

import oracle as O
import paper_2501_07642_b200 as frr
from paper_2501_07642_b200.errors import InvalidDesignError

pytestmark = pytest.mark.gpu
M64 = (1 << 64) - 1


def unpack(bits, n):
    return np.unpackbits(bits, axis=1, count=n, bitorder="little").astype(np.int8)


@pytest.mark.parametrize("case", range(9))
def test_golden_assignments(golden, case):
    g = golden("keys")
    n, t = (int(v) for v in g["cases"][case])
    for si, s in enumerate(g["seeds"]):
        got = frr.batch_assignments(int(s), g["draws"], n, t)
        assert np.array_equal(got, unpack(g[f"bits_{n}_{t}_{si}"], n)), (n, t, si)


def test_known_answer_and_scalar_path(golden):
    a = frr.assignment_from_key(frr.AssignmentKey(7, 0), 20, 10)
    assert np.flatnonzero(a.bits).tolist() == [1, 2, 4, 5, 7, 8, 9, 10, 12, 14]
    assert a.n_treated == 10 and a.n_units == 20


@pytest.mark.parametrize("n,t", [(2, 1), (3, 2), (17, 8), (100, 1), (100, 99), (1000, 500), (4097, 2000),
                                 (5000, 2500), (40000, 20000),
                                 # t close to a multiple-of-32 n: padding steps re-read past the table
                                 (64, 63), (1024, 1023), (1056, 1055)])
def test_random_draws_vs_oracle(n, t):
    rng = np.random.default_rng(n + t)
    m = 2000 if n <= 5000 else 64
    draws = rng.integers(0, 2**63, size=m, dtype=np.int64).astype(np.uint64) * np.uint64(2)
    draws[:3] = [0, 1, M64]
    seed = int(rng.integers(0, 2**63)) * 2 + 1
    assert np.array_equal(frr.batch_assignments(seed, draws, n, t), O.c_batch_assign(seed, draws, n, t))


def test_bits_output_matches_rows():
    import torch

    from paper_2501_07642_b200 import keys as K

    draws = K.to_device_u64(np.arange(777, dtype=np.uint64) * np.uint64(3))
    rows = K.regen_rows_device(11, draws, 1000, 321).cpu().numpy()
    bits = K.regen_bits_device(11, draws, 1000, 321).cpu().numpy().view(np.uint32)
    unpacked = np.unpackbits(bits.view(np.uint8), axis=1, bitorder="little")[:, :1000].astype(np.int8)
    assert np.array_equal(unpacked, rows)
    assert (rows.sum(axis=1) == 321).all()
    torch.cuda.synchronize()


def test_subset_order_independence_and_empty():
    all_rows = frr.batch_assignments(1, np.arange(50, dtype=np.uint64), 6, 3)
    subset = frr.batch_assignments(1, np.array([44, 3, 17], dtype=np.uint64), 6, 3)
    assert np.array_equal(subset, all_rows[[44, 3, 17]])
    assert frr.batch_assignments(1, np.array([], dtype=np.uint64), 6, 3).shape == (0, 6)


def test_uniformity_small_design():
    scipy_stats = pytest.importorskip("scipy.stats")
    batch = frr.batch_assignments(2024, np.arange(60_000, dtype=np.uint64), 4, 2)
    codes = batch @ (1 << np.arange(4))
    _, counts = np.unique(codes, return_counts=True)
    assert counts.shape[0] == 6
    chi2 = float(((counts - 10_000) ** 2 / 10_000).sum())
    assert scipy_stats.chi2.sf(chi2, df=5) > 0.001


@pytest.mark.parametrize("n,t", [(10, 0), (10, 10), (1, 1)])
def test_invalid(n, t):
    with pytest.raises(InvalidDesignError):
        frr.batch_assignments(0, np.arange(3, dtype=np.uint64), n, t)
    with pytest.raises(InvalidDesignError):
        frr.batch_assignments(5, np.array([-1]), 6, 3)


REJ_CASES = range(9)


@pytest.mark.parametrize("case", REJ_CASES)
def test_rejection_keys_golden(golden, case):
    """The GPU generator's exact sequential path (taken when a stream output
    has hi(u) == 0xFFFFFFFF) against the reference, for keys crafted to be
    rejected at a chosen step (first, middle, last) or only flagged."""
    g = golden("rejection")
    n, t, _ = (int(v) for v in g["cases"][case])
    seed, draw = int(g["seeds"][case]), int(g["draw"])
    draws = np.array([draw, draw + 1, 0], dtype=np.uint64)
    assert np.array_equal(frr.batch_assignments(seed, draws, n, t), unpack(g[f"bits_{case}"], n))


@pytest.mark.parametrize("n,t", [(2, 1), (20, 10), (34, 17), (33, 1), (40, 39), (64, 32), (64, 3), (66, 33)])
def test_exact_rows_vs_oracle(n, t):
    """Accepted-rank regeneration (frr_regen_exact: thread-per-rank rows for
    n <= 64, the warp path above) against the oracle's combinadic unranking."""
    import math

    from paper_2501_07642_b200 import generation as G

    total = math.comb(n, t)
    rng = np.random.default_rng(n * 7 + t)
    m = min(total, 5001)
    hi = min(total, 2**62)
    ranks = np.unique(np.concatenate([np.array([0, hi - 1], dtype=np.uint64),
                                      rng.integers(0, hi, size=m, dtype=np.uint64)]))
    got = G.exact_rows_device(ranks, n, t).cpu().numpy()
    assert np.array_equal(got, O.c_exact_rows(ranks, n, t))
