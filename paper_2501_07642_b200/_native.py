"""ctypes binding of libfrr.so (include/frr.h) -- the only path to compute.

The CUDA library is mandatory: there is no CPU fallback.  Importing the
package works without a GPU (so host-only helpers and validation can be
used and tested), but every compute entry point raises
:class:`~paper_2501_07642_b200.errors.NativeUnavailableError` when
libfrr.so or a CUDA device is missing.
"""

from __future__ import annotations

import ctypes
import os
import threading

from . import errors as E

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FRR_LIBRARY", os.path.join(_HERE, "libfrr.so"))
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "frr.h")

FRR_OK = 0
_CODE_TO_ERROR = {
    1: E.InvalidDesignError,
    2: E.DimensionError,
    3: E.EnumerationTooLargeError,
    4: E.StorageCapError,
    5: E.UnsupportedShapeError,
    64: E.DeviceError,
}

u64, i64, i32, dbl, vp, sz = (ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, ctypes.c_double,
                              ctypes.c_void_p, ctypes.c_size_t)


class Balance(ctypes.Structure):
    """Mirror of ``frr_balance_t``."""

    _fields_ = [
        ("n", ctypes.c_int32), ("d", ctypes.c_int32), ("t", ctypes.c_int32), ("n_limbs", ctypes.c_int32),
        ("zq", vp), ("colsum", vp), ("cc", vp), ("limbs", vp),
        ("g", dbl), ("cst", dbl),
    ]


SIGNATURES = {
    "frr_abi_version": (i32, []),
    "frr_last_error": (ctypes.c_char_p, []),
    "frr_device_info": (i32, [ctypes.POINTER(i32)] * 3),
    "frr_tc_kernel": (i32, [i32, i32, i32]),
    "frr_limbs_bytes": (sz, [i32, i32, i32]),
    "frr_prepare_limbs": (i32, [vp, i32, i32, i32, vp, vp, vp]),
    "frr_mc_stats": (i32, [ctypes.POINTER(Balance), u64, u64, i64, vp, vp]),
    "frr_mc_stats_small": (i32, [ctypes.POINTER(Balance), u64, u64, i64, vp, vp]),
    "frr_mc_stats_tc": (i32, [ctypes.POINTER(Balance), u64, u64, i64, vp, vp]),
    "frr_exact_stats": (i32, [ctypes.POINTER(Balance), u64, i64, vp, vp]),
    "frr_exact_stats_ids": (i32, [ctypes.POINTER(Balance), vp, i64, vp, vp]),
    "frr_exact_split_width": (i32, [i32]),
    "frr_subset_sums": (i32, [ctypes.POINTER(Balance), i32, i32, vp, vp, vp, vp]),
    "frr_exact_stats_split": (i32, [ctypes.POINTER(Balance), vp, vp, i32, vp, vp, vp, i64, u64, i64, vp, vp]),
    "frr_exact_stats_split_strided": (i32, [ctypes.POINTER(Balance), vp, vp, i32, vp, vp, vp, i64, u64, i64, i64,
                                            vp, vp]),
    "frr_exact_tiled_filtered": (i32, [ctypes.POINTER(Balance), vp, vp, i32, vp, i64, vp, vp, u64, u64, u64, i64,
                                       vp, vp, vp, vp]),
    "frr_exact_stats_split_filtered": (i32, [ctypes.POINTER(Balance), vp, vp, i32, vp, vp, vp, i64, u64, i64, u64,
                                             i64, vp, vp, vp, vp]),
    "frr_rows_stats": (i32, [ctypes.POINTER(Balance), vp, i64, vp, vp]),
    "frr_regen_mc": (i32, [u64, vp, i64, i32, i32, vp, vp, vp]),
    "frr_regen_exact": (i32, [vp, i64, i32, i32, vp, vp, vp]),
    "frr_select_init": (i32, [vp, i64, vp]),
    "frr_select_hist": (i32, [vp, i64, vp, i32, vp, vp]),
    "frr_select_pick": (i32, [vp, vp, i32, vp]),
    "frr_select_count": (i32, [vp, i64, vp, vp, vp]),
    "frr_select_workspace_bytes": (sz, [i64]),
    "frr_select_compact": (i32, [vp, i64, i64, vp, vp, vp, vp, vp, vp, vp]),
    "frr_select_compact_capped": (i32, [vp, i64, i64, vp, vp, i64, vp, vp, vp, vp, vp]),
    "frr_sort_pairs_workspace_bytes": (sz, [i64]),
    "frr_sort_pairs": (i32, [vp, vp, i64, i32, vp, sz, vp]),
    "frr_dim_mc": (i32, [u64, vp, i64, i32, i32, vp, vp, vp, vp, vp, vp]),
    "frr_dim_mc_workspace_bytes": (sz, [i64, i32]),
    "frr_dim_mc_chunk_keys": (i64, [i64, i32, i32, sz]),
    "frr_dim_mc_ws": (i32, [u64, vp, i64, i32, i32, vp, vp, vp, vp, vp, vp, sz, vp]),
    "frr_dim_exact": (i32, [vp, i64, i32, i32, vp, vp, vp, vp, vp, vp]),
    "frr_dim_rows": (i32, [vp, i64, i32, i32, vp, vp, vp, vp, vp, vp]),
    "frr_tau_counts": (i32, [vp, vp, i64, vp, vp, i32, vp, vp]),
    "frr_selftest_mma_i8": (i32, [vp, vp, i32, i32, vp, i32, vp]),
    "frr_microbench_draws": (i32, [i64, vp, vp, vp]),
    "frr_microbench_mma_i8": (i32, [i32, i32, i64, vp, vp]),
    "frr_microbench_mma_i8_pair": (i32, [i32, i32, i64, vp, vp]),
    "frr_rev_bits": (i32, [u64, u64, i64, i32, i32, vp, vp, vp]),
    "frr_launch_count": (ctypes.c_ulonglong, []),
    "frr_sim_pairs": (i32, [u64, u64, i64, i64, vp, vp, vp, vp]),
}

_lock = threading.Lock()
_lib = None


def load_library(path: str | None = None) -> ctypes.CDLL:
    """Load libfrr.so and bind every exported symbol (no device needed)."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise E.NativeUnavailableError(
                f"libfrr.so not found at {p}; build it with `python __graft_entry__.py` "
                "(make -C paper_2501_07642_b200/csrc)")
        lib = ctypes.CDLL(p)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.frr_abi_version() != 1:
            raise E.NativeUnavailableError("libfrr.so ABI version mismatch")
        if path is None:
            _lib = lib
        return lib


def lib() -> ctypes.CDLL:
    return _lib if _lib is not None else load_library()


_torch = None


def torch_mod():
    global _torch
    if _torch is None:
        import torch

        _torch = torch
    return _torch


def device():
    """The CUDA device compute runs on (current device); fails loudly."""
    torch = torch_mod()
    if not torch.cuda.is_available():
        raise E.NativeUnavailableError(
            "no CUDA device: the rerandomization engine runs only on the GPU (no CPU fallback)")
    lib()
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr():
    torch = torch_mod()
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def check(rc: int, what: str):
    if rc != FRR_OK:
        msg = lib().frr_last_error().decode(errors="replace")
        cls = _CODE_TO_ERROR.get(rc, E.DeviceError)
        raise cls(f"{what}: {msg}")


def call(name: str, *args):
    check(getattr(lib(), name)(*args), name)



STAGE_MIN_BYTES = 1 << 20
STAGE_CHUNK = 4 << 20  # bytes per page-locked staging slot
STAGE_SLOTS = 16       # slots in the ring (64 MB of page-locked host memory in all)
_stage_lock = threading.Lock()
_stage = {"ring": None, "pool": None}


def _stage_ring():
    torch = torch_mod()
    if _stage["ring"] is None:
        _stage["ring"] = [torch.empty(STAGE_CHUNK, dtype=torch.uint8, pin_memory=True) for _ in range(STAGE_SLOTS)]
    return _stage["ring"]


def to_host(t):
    """Device tensor -> a numpy array the caller owns; see to_host_many."""
    return to_host_many(t)[0]


# Recycled page-locked result buffers.  A large result is copied by one DMA
# straight into a page-locked slab that the caller's numpy array views; when
# the last view of that array dies, the slab returns to the pool for the next
# result (PEP 688 buffer release), so repeated calls neither page-lock nor
# first-touch (~10 GB/s of page faults) new memory.  The pool is bounded:
# FRR_HOST_POOL_MB (default 1024; 0 disables) of page-locked memory at most,
# beyond which results go through the staging ring below.
HOST_POOL_BYTES = int(os.environ.get("FRR_HOST_POOL_MB", "1024")) << 20
HOST_POOL_ALIGN = 2 << 20
_pool_lock = threading.Lock()
_pool = {"free": [], "bytes": 0}


class _PooledResult:
    """Buffer exporter of one result: a byte range of a pooled slab.  The
    slab goes back to the pool when the last exported view is released."""

    __slots__ = ("slab", "nbytes", "views")

    def __init__(self, slab, nbytes):
        self.slab = slab
        self.nbytes = nbytes
        self.views = 0

    def __buffer__(self, flags):
        if self.slab is None:
            raise BufferError("pooled result already released")
        self.views += 1
        return memoryview(self.slab.numpy()[: self.nbytes])

    def __release_buffer__(self, view):
        view.release()
        self.views -= 1
        if self.views == 0 and self.slab is not None:
            slab, self.slab = self.slab, None
            with _pool_lock:
                _pool["free"].append(slab)


def _pool_take(nbytes):
    """A free slab of at least nbytes (best fit within 2x), a new one while
    the pool is under its bound, or None."""
    torch = torch_mod()
    with _pool_lock:
        free = _pool["free"]
        fits = [i for i, s in enumerate(free) if nbytes <= s.numel() <= 2 * nbytes + HOST_POOL_ALIGN]
        if fits:
            i = min(fits, key=lambda i: free[i].numel())
            return free.pop(i)
        size = -(-nbytes // HOST_POOL_ALIGN) * HOST_POOL_ALIGN
        if _pool["bytes"] + size > HOST_POOL_BYTES:
            return None
        _pool["bytes"] += size
    return torch.empty(size, dtype=torch.uint8, pin_memory=True)


def _np_dtype(t):
    torch = torch_mod()
    return torch.empty(0, dtype=t.dtype).numpy().dtype


def to_host_many(*tensors):
    """Device tensors -> numpy arrays the caller owns.  Large results
    (accepted indices, statistics, assignment rows) are DMA'd into recycled
    page-locked slabs (above) that the returned arrays view, all on one
    stream with one synchronisation.  Results that do not fit the pool's
    bound stream through a fixed ring of page-locked staging slots into fresh
    numpy arrays: the DMA of chunk i + 1 overlaps the host copy of chunk i out
    of its slot (a pageable .cpu() of the 79 MB C4 row matrix runs at
    ~2 GB/s)."""
    torch = torch_mod()
    import numpy as np

    outs = [None] * len(tensors)
    big = []
    dma = None
    for i, t in enumerate(tensors):
        nbytes = t.numel() * t.element_size()
        if not t.is_cuda or nbytes < STAGE_MIN_BYTES:
            outs[i] = t.cpu().numpy()
            continue
        slab = _pool_take(nbytes)
        if slab is None:
            big.append(i)
            continue
        t = t.contiguous()
        slab[:nbytes].copy_(t.reshape(-1).view(torch.uint8), non_blocking=True)
        outs[i] = np.frombuffer(_PooledResult(slab, nbytes), dtype=_np_dtype(t)).reshape(tuple(t.shape))
        dma = torch.cuda.current_stream(t.device)
    if dma is not None:
        dma.synchronize()
    if not big:
        return outs
    from concurrent.futures import ThreadPoolExecutor

    with _stage_lock:
        ring = _stage_ring()
        if _stage["pool"] is None:
            # host copies of different slots run in parallel (np.copyto drops the GIL)
            _stage["pool"] = ThreadPoolExecutor(max(1, min(8, os.cpu_count() or 1)))
        pending = [None] * STAGE_SLOTS  # host-copy future per slot

        def land(slot, dst, a, n, ev):
            ev.synchronize()
            np.copyto(dst[a:a + n], ring[slot].numpy()[:n])

        k = 0
        for i in big:
            t = tensors[i].contiguous()
            out = np.empty(tuple(t.shape), dtype=_np_dtype(t))
            outs[i] = out
            dst = out.reshape(-1).view(np.uint8)
            flat = t.reshape(-1).view(torch.uint8)
            nbytes = flat.numel()
            stream = torch.cuda.current_stream(t.device)
            for a in range(0, nbytes, STAGE_CHUNK):
                slot = k % STAGE_SLOTS
                k += 1
                if pending[slot] is not None:
                    pending[slot].result()  # the slot's previous chunk has left it
                n = min(STAGE_CHUNK, nbytes - a)
                ring[slot][:n].copy_(flat[a:a + n], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(stream)
                pending[slot] = _stage["pool"].submit(land, slot, dst, a, n, ev)
        for f in pending:
            if f is not None:
                f.result()
    return outs
    from concurrent.futures import ThreadPoolExecutor

    with _stage_lock:
        ring = _stage_ring()
        if _stage["pool"] is None:
            # host copies of different slots run in parallel (np.copyto drops the GIL)
            _stage["pool"] = ThreadPoolExecutor(max(1, min(8, os.cpu_count() or 1)))
        pending = [None] * STAGE_SLOTS  # host-copy future per slot

        def land(slot, dst, a, n, ev):
            ev.synchronize()
            np.copyto(dst[a:a + n], ring[slot].numpy()[:n])

        k = 0
        for i in big:
            t = tensors[i].contiguous()
            out = np.empty(tuple(t.shape), dtype=torch.empty(0, dtype=t.dtype).numpy().dtype)
            outs[i] = out
            dst = out.reshape(-1).view(np.uint8)
            flat = t.reshape(-1).view(torch.uint8)
            nbytes = flat.numel()
            stream = torch.cuda.current_stream(t.device)
            for a in range(0, nbytes, STAGE_CHUNK):
                slot = k % STAGE_SLOTS
                k += 1
                if pending[slot] is not None:
                    pending[slot].result()  # the slot's previous chunk has left it
                n = min(STAGE_CHUNK, nbytes - a)
                ring[slot][:n].copy_(flat[a:a + n], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(stream)
                pending[slot] = _stage["pool"].submit(land, slot, dst, a, n, ev)
        for f in pending:
            if f is not None:
                f.result()
    return outs
