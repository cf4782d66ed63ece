"""Pool files and threshold sweeps against the reference's own outputs
(tests/golden/poolio.npz, sweep.npz, written by oracle/make_golden.py from
the reference fastrr 0.1.0): byte-identical CSV pool files for Monte Carlo
keys / full / both storage (streamed with out_path and written with
write_pool) and exact pools (streamed and written), read_pool's parse of
each reference file, and the sweep rows (p-values, pool sizes, interval
widths, the failure status of failing rows) -- SURVEY section 8 f1, f2."""

import dataclasses
import hashlib
import json

import numpy as np
import pytest

import paper_2501_07642_b200 as frr
from paper_2501_07642_b200 import generation as G

pytestmark = pytest.mark.gpu

MC_X = np.random.default_rng(301).standard_normal((40, 3))
MC_BASE = frr.DesignSpec(n_units=40, n_treated=20, accept_prob=0.01, max_draws=3000, batch_size=257,
                         root_seed=301, precision_mode="exact")
EX_X = np.random.default_rng(302).standard_normal((12, 3))
EX_DESIGN = frr.DesignSpec(n_units=12, n_treated=6, accept_prob=0.05, mode="exact", batch_size=100)


def _bytes(path):
    with open(path, "rb") as f:
        return f.read()


@pytest.mark.parametrize("storage", ["keys", "full", "both"])
def test_mc_pool_files_byte_identical(golden, tmp_path, storage):
    g = golden("poolio")
    design = dataclasses.replace(MC_BASE, storage=storage)
    path = tmp_path / "stream.csv"
    frr.generate_pool(MC_X, design, workers=1, out_path=path)
    assert _bytes(path) == g[f"mc_{storage}_stream"].tobytes()
    pool = frr.generate_pool(MC_X, design, workers=1)
    path = tmp_path / "write.csv"
    frr.write_pool(pool, path)
    assert _bytes(path) == g[f"mc_{storage}_write"].tobytes()


def test_exact_pool_files_byte_identical(golden, tmp_path):
    g = golden("poolio")
    path = tmp_path / "stream.csv"
    frr.generate_pool(EX_X, EX_DESIGN, out_path=path)
    assert _bytes(path) == g["exact_stream"].tobytes()
    pool = frr.generate_pool(EX_X, EX_DESIGN)
    path = tmp_path / "write.csv"
    frr.write_pool(pool, path)
    assert _bytes(path) == g["exact_write"].tobytes()


@pytest.mark.parametrize("name", ["mc_keys_stream", "mc_full_write", "mc_both_stream", "exact_stream",
                                  "exact_write"])
def test_read_reference_pool_file(golden, tmp_path, name):
    g = golden("poolio")
    path = tmp_path / "ref.csv"
    path.write_bytes(g[name].tobytes())
    rp = frr.read_pool(path)
    want = json.loads(g[f"read_{name}"].tobytes())
    assert rp.design.to_json_dict() == want["design"]
    assert rp.threshold_value == want["threshold"] and rp.n_candidates == want["n_candidates"]
    assert [repr(float(v)) for v in rp.stats] == want["stats"]
    got_acc = None if rp.accepted_indices is None else [int(v) for v in rp.accepted_indices]
    assert got_acc == want["accepted"]
    assert (None if rp.keys is None else [[int(a), int(b)] for a, b in rp.keys]) == want["keys"]
    sha = None if rp.assignments is None else hashlib.sha256(
        np.ascontiguousarray(rp.assignments.astype(np.int8)).tobytes()).hexdigest()
    assert sha == want["assignments_sha"]
    # and a pool read back from the reference's file tests like the in-memory one
    if rp.keys is not None or rp.assignments is not None:
        mat = frr.pool_assignment_matrix(rp)
        y = np.arange(mat.shape[1], dtype=np.float64)
        res = frr.randomization_test(mat[0], y, rp)
        assert 0.0 < res.p_value <= 1.0


def _rows(raw):
    return [{k: (repr(v) if isinstance(v, float) else v) for k, v in r.items()} for r in raw]


@pytest.mark.parametrize("find_fi", [False, True])
def test_threshold_sweep_rows_match_reference(golden, find_fi):
    g = golden("sweep")
    X = np.random.default_rng(311).standard_normal((30, 3))
    rng = np.random.default_rng(312)
    y = X @ rng.standard_normal(3) + 0.5 * rng.standard_normal(30)
    base = frr.DesignSpec(n_units=30, n_treated=15, accept_prob=0.1, max_draws=4000, batch_size=500,
                          root_seed=311, precision_mode="exact")
    rows = frr.threshold_sweep(X, base, list(g["probs"]), y, find_fi=find_fi, alpha=0.1, workers=1)
    assert _rows(rows) == json.loads(g[f"rows_fi{int(find_fi)}"].tobytes())


def test_threshold_sweep_exact_rows_match_reference(golden):
    g = golden("sweep")
    Xe = np.random.default_rng(313).standard_normal((12, 3))
    ye = Xe[:, 0] + 0.3 * np.random.default_rng(314).standard_normal(12)
    exb = frr.DesignSpec(n_units=12, n_treated=6, accept_prob=0.1, mode="exact")
    rows = frr.threshold_sweep(Xe, exb, [0.5, 0.2, 0.05, 0.01], ye, find_fi=True, alpha=0.2)
    assert _rows(rows) == json.loads(g["rows_exact"].tobytes())


def test_streamed_exact_pool_then_test_raises_reference_error(tmp_path):
    """An exact pool streamed to a file keeps neither keys nor assignments in
    memory; testing it raises the reference's InvalidDesignError
    (generation.py:349-352 via pool_assignment_matrix)."""
    pool = frr.generate_pool(EX_X, EX_DESIGN, out_path=tmp_path / "p.csv")
    assert pool.keys is None and pool.assignments is None
    with pytest.raises(frr.errors.InvalidDesignError, match="pool stores no keys"):
        frr.randomization_test(np.r_[np.ones(6), np.zeros(6)].astype(np.int8), np.arange(12.0), pool)
    with pytest.raises(frr.errors.InvalidDesignError, match="pool stores no keys"):
        G.pool_assignment_matrix(pool)
