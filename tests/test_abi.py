"""C-ABI boundary and host-side logic -- CPU only (no compute calls)."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2501_07642_b200 as frr
from paper_2501_07642_b200 import _native as N
from paper_2501_07642_b200 import errors as E
from paper_2501_07642_b200.balance import _n_limbs
from paper_2501_07642_b200.inference import _pack_bits

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "frr.h")).read()
    return sorted(set(re.findall(r"^\s*(?:[A-Za-z_][\w ]*[\s\*])(frr_\w+)\s*\(", src, flags=re.M)))


def test_library_loads_and_exports_every_header_symbol():
    lib = N.load_library()
    names = header_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
        assert name in N.SIGNATURES, f"{name} not bound in _native.SIGNATURES"
    assert lib.frr_abi_version() == 1


def test_library_is_sm100a():
    so = N.LIB_PATH
    out = os.popen(f"cuobjdump -lelf {so} 2>/dev/null").read()
    assert "sm_100a" in out


def test_status_codes_map_to_reference_error_codes():
    assert E.InvalidDesignError.code == "invalid_design"
    assert E.DimensionError.code == "dimension_mismatch"
    assert E.EnumerationTooLargeError.code == "enumeration_too_large"
    assert E.StorageCapError.code == "storage_cap_exceeded"
    assert N._CODE_TO_ERROR[1] is E.InvalidDesignError
    assert N._CODE_TO_ERROR[3] is E.EnumerationTooLargeError


def test_balance_struct_layout_matches_header():
    assert ctypes.sizeof(N.Balance) == 4 * 4 + 4 * 8 + 2 * 8


def test_limbs_bytes_c2():
    lib = N.load_library()
    # n=1000 -> K padded to 1024; 6 limbs x d=64 -> N=384
    assert lib.frr_limbs_bytes(1000, 64, 6) == 1024 * 384


def test_tc_kernel_choice():
    lib = N.load_library()
    assert lib.frr_tc_kernel(1000, 64, 6) == 1      # C2: single pass, N = 384 columns
    assert lib.frr_tc_kernel(2000, 1024, 6) == 2    # C3: N-tiled
    assert lib.frr_tc_kernel(20, 100, 7) == 2       # 7 limbs: N-tiled with 128-byte K stages
    assert lib.frr_tc_kernel(34, 5, 7) == 0         # d <= 16: CUDA-core warp kernel
    assert lib.frr_tc_kernel(8200, 96, 6) == 0      # bit rows of n=8200 do not fit shared memory
    assert lib.frr_tc_kernel(5000, 128, 6) == 2     # large n: N-tiled with one bit buffer
    # the N-tiled operand: 32-covariate chunks x 2048 K bytes x 6*32 rows
    assert lib.frr_limbs_bytes(2000, 1024, 6) == 32 * 2048 * 192


@pytest.mark.parametrize("n,t", [(10, 0), (10, 10), (10, 11), (1, 1)])
def test_invalid_designs(n, t):
    with pytest.raises(E.InvalidDesignError):
        frr.DesignSpec(n_units=n, n_treated=t)


def test_design_validation_rules():
    with pytest.raises(E.InvalidDesignError):
        frr.DesignSpec(10, 5, accept_prob=0.0)
    with pytest.raises(E.InvalidDesignError):
        frr.DesignSpec(10, 5, max_draws=0)
    with pytest.raises(E.InvalidDesignError):
        frr.DesignSpec(10, 5, max_draws=10, batch_size=11)
    with pytest.raises(E.InvalidDesignError):
        frr.DesignSpec(10, 5, mode="bogus")
    with pytest.raises(E.InvalidDesignError):
        frr.DesignSpec(10, 5, ridge_scale=0.0)
    with pytest.raises(E.EnumerationTooLargeError):
        frr.DesignSpec(200, 100, mode="exact").n_exact_candidates()


def test_key_wire_format_and_scalar_contract():
    key = frr.AssignmentKey(0x0102030405060708, 3)
    raw = key.to_bytes()
    assert raw[:8] == bytes([8, 7, 6, 5, 4, 3, 2, 1]) and raw[8:] == bytes([3] + [0] * 7)
    assert frr.AssignmentKey.from_bytes(raw) == key
    assert frr.derive_state(frr.AssignmentKey(0, 0)) == 0xE220A8397B1DCDAF
    with pytest.raises(E.InvalidDesignError):
        frr.AssignmentKey(-1, 0)
    assert frr.memory_improvement_factor(1000, 2) == 500


def test_pack_bits_layout():
    w = np.zeros(70, dtype=np.int8)
    w[[0, 5, 31, 32, 69]] = 1
    b = _pack_bits(w)
    assert b.dtype == np.uint32 and b.shape == (3,)
    assert b[0] == (1 | (1 << 5) | (1 << 31)) and b[1] == 1 and b[2] == (1 << 5)


def test_limb_count():
    assert _n_limbs(np.array([0.0])) == 1
    assert _n_limbs(np.array([127.0, -128.0])) == 1
    assert _n_limbs(np.array([128.0])) == 2
    assert _n_limbs(np.array([2.0**46 - 1, -(2.0**46)])) == 6


def test_compute_fails_loudly_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(E.NativeUnavailableError):
        frr.batch_assignments(1, np.arange(3), 10, 5)


def test_pool_file_round_trip_keys_storage(tmp_path):
    design = frr.DesignSpec(12, 6, accept_prob=0.5, max_draws=6, batch_size=6, root_seed=77)
    pool = frr.RandomizationPool(design=design, stats=np.array([0.1, 0.25, 1 / 3]), threshold_value=1 / 3,
                                 n_candidates=6, accepted_indices=np.array([0, 2, 5]),
                                 keys=np.column_stack([np.full(3, 77, dtype=np.uint64),
                                                       np.array([0, 2, 5], dtype=np.uint64)]))
    path = tmp_path / "p.csv"
    frr.write_pool(pool, path)
    text = path.read_text().splitlines()
    assert text[0] == "# fastrr-pool v1" and text[2] == "key_seed,key_draw,stat"
    assert text[3] == "77,0,0.1"
    back = frr.read_pool(path)
    assert np.array_equal(back.stats, pool.stats) and np.array_equal(back.keys, pool.keys)
    assert back.threshold_value == pool.threshold_value
    bad = tmp_path / "bad.csv"
    bad.write_text("# fastrr-pool v1\n# wrong header\nstat\n")
    with pytest.raises(E.PoolFormatError):
        frr.read_pool(bad)


def test_pool_summary_arithmetic():
    design = frr.DesignSpec(12, 6, accept_prob=0.5, max_draws=6, batch_size=6)
    pool = frr.RandomizationPool(design=design, stats=np.array([0.1, 0.2, 0.3]), threshold_value=0.3,
                                 n_candidates=6, accepted_indices=np.array([0, 1, 2]))
    s = frr.pool_summary(pool)
    assert s["stat_min"] == pytest.approx(0.1) and s["stat_median"] == pytest.approx(0.2)
    assert s["acceptance_rate"] == pytest.approx(0.5)


def test_public_surface_matches_reference_names():
    for name in ["generate_pool", "monte_carlo_pool", "enumerate_exact", "regenerate_assignments",
                 "pool_assignment_matrix", "batch_assignments", "batch_balance", "randomization_pvalue",
                 "fiducial_interval", "randomization_test", "DesignSpec", "RandomizationPool", "TestResult",
                 "generate_randomizations", "threshold_sweep", "precompute_precision", "mahalanobis_stat"]:
        assert hasattr(frr, name), name
    from paper_2501_07642_b200.generation import _resolve_workers, pools_equal  # noqa: F401
    from paper_2501_07642_b200.keys import GOLDEN, MASK64, mix64  # noqa: F401
