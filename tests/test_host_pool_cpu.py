"""The recycled result slabs' exporter logic (_native._PooledResult) on CPU:
the slab returns to the pool only when the last exported view is released,
and a released handle cannot be exported again."""
import gc

import numpy as np
import pytest

from paper_2501_07642_b200 import _native as N


class _Slab:  # stand-in for a page-locked torch tensor
    def __init__(self, n):
        self.a = np.arange(n, dtype=np.uint8)

    def numpy(self):
        return self.a

    def numel(self):
        return self.a.size


def test_slab_returns_after_last_view():
    before = len(N._pool["free"])
    h = N._PooledResult(_Slab(64), 48)
    arr = np.frombuffer(h, dtype=np.int64)
    assert arr.shape == (6,) and arr.flags.writeable
    view = arr[2:4]
    extra = memoryview(h)
    del arr
    gc.collect()
    assert len(N._pool["free"]) == before
    del view
    gc.collect()
    assert len(N._pool["free"]) == before  # `extra` still exports the slab
    extra.release()
    gc.collect()
    assert len(N._pool["free"]) == before + 1
    N._pool["free"].pop()
    with pytest.raises(BufferError):
        memoryview(h)
