"""Recycled page-locked result buffers of _native.to_host_many: values,
recycling when the caller's arrays die, the pool bound and the staging-ring
fall-back."""
import gc

import numpy as np
import pytest
import torch

from paper_2501_07642_b200 import _native as N

pytestmark = pytest.mark.gpu


def _tensors(seed, m=300_000):
    g = torch.Generator(device="cuda").manual_seed(seed)
    rows = torch.randint(-1, 2, (m, 34), dtype=torch.int8, device="cuda", generator=g)
    idx = torch.randint(0, 1 << 40, (m,), dtype=torch.int64, device="cuda", generator=g)
    st = torch.rand(m, dtype=torch.float64, device="cuda", generator=g)
    return rows, idx, st


def test_values_and_recycling():
    rows, idx, st = _tensors(1)
    a, b, c = N.to_host_many(idx, st, rows)
    np.testing.assert_array_equal(a, idx.cpu().numpy())
    np.testing.assert_array_equal(b, st.cpu().numpy())
    np.testing.assert_array_equal(c, rows.cpu().numpy())
    assert c.shape == (300_000, 34) and c.dtype == np.int8 and c.flags.writeable
    c[0, 0] = 7  # caller-owned: writable
    view = c[10:20]
    free_before = len(N._pool["free"])
    del a, b, c
    gc.collect()
    # the row slab stays out of the pool while a view of it lives
    assert len(N._pool["free"]) == free_before + 2
    del view
    gc.collect()
    assert len(N._pool["free"]) == free_before + 3
    # the next results reuse those slabs: no new page-locked memory
    total = N._pool["bytes"]
    rows2, idx2, st2 = _tensors(2)
    a2, b2, c2 = N.to_host_many(idx2, st2, rows2)
    assert N._pool["bytes"] == total
    np.testing.assert_array_equal(c2, rows2.cpu().numpy())
    np.testing.assert_array_equal(a2, idx2.cpu().numpy())


def test_bound_falls_back_to_staging(monkeypatch):
    rows, idx, st = _tensors(3)
    monkeypatch.setattr(N, "HOST_POOL_BYTES", N._pool["bytes"])  # no room for new slabs
    keep = [N.to_host_many(rows) for _ in range(4)]  # more live results than free slabs
    for (r,) in keep:
        np.testing.assert_array_equal(r, rows.cpu().numpy())
    assert N._pool["bytes"] <= N.HOST_POOL_BYTES
