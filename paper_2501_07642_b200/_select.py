"""Exact acceptance selection (generation.py:159-169) on device, 1..N GPUs.

``select_k_smallest`` is the orchestration: an 8-pass MSD radix select over
the statistics' IEEE bit patterns (statistics are >= +0, so bit order is
value order) with the per-pass 256-bin histogram all-reduced across ranks,
then a tie quota split in rank (= index) order, an order-preserving local
compaction and a rank-ordered gather.  The result equals the reference's
stable argsort rule: the k smallest by (stat, index), returned ascending
by index, with threshold = the k-th smallest stat.

The local operations come from an ``ops`` object (``DeviceSelectOps`` here,
backed by libfrr kernels); the collective from a ``comm`` object
(``TorchComm`` over torch.distributed -- NCCL on the GPU path).  Candidates
are sharded by contiguous index range, so the only collectives are the
histogram all-reduce (8 x 2 KB), one all-gather of two counts, and the
accepted-key gather.
"""

from __future__ import annotations

import numpy as np

from . import _native as N


class DeviceSelectOps:
    """Local select steps as libfrr kernels on the current CUDA stream."""

    def __init__(self):
        self.torch = N.torch_mod()

    def init(self, k: int, device):
        st = self.torch.empty(4, dtype=self.torch.int64, device=device)
        N.call("frr_select_init", N.ptr(st), int(k), N.stream_ptr())
        return st

    def hist(self, stats, st, p: int):
        h = self.torch.empty(256, dtype=self.torch.int64, device=st.device)
        N.call("frr_select_hist", N.ptr(stats), int(stats.shape[0]), N.ptr(st), p, N.ptr(h), N.stream_ptr())
        return h

    def pick(self, hist, st, p: int):
        N.call("frr_select_pick", N.ptr(hist), N.ptr(st), p, N.stream_ptr())

    def counts(self, stats, st):
        c = self.torch.empty(2, dtype=self.torch.int64, device=st.device)
        N.call("frr_select_count", N.ptr(stats), int(stats.shape[0]), N.ptr(st), N.ptr(c), N.stream_ptr())
        return c

    def k_rem(self, st):
        return st[2:3]

    def compact(self, stats, index_base: int, st, quota, cap: int):
        torch = self.torch
        m = int(stats.shape[0])
        cap = max(1, min(int(cap), m))
        idx = torch.empty(cap, dtype=torch.int64, device=st.device)
        val = torch.empty(cap, dtype=torch.float64, device=st.device)
        n_out = torch.empty(1, dtype=torch.int64, device=st.device)
        ws = torch.empty(int(N.lib().frr_select_workspace_bytes(m)) // 8 + 1, dtype=torch.int64, device=st.device)
        N.call("frr_select_compact", N.ptr(stats), m, int(index_base), N.ptr(st), N.ptr(quota), N.ptr(idx),
               N.ptr(val), N.ptr(n_out), N.ptr(ws), N.stream_ptr())
        return idx, val, n_out

    def threshold(self, st) -> float:
        bits = int(st[0].item()) & ((1 << 64) - 1)
        return float(np.array([bits], dtype=np.uint64).view(np.float64)[0])


class LocalComm:
    rank, world = 0, 1

    def all_reduce_(self, t):
        return t

    def all_gather(self, t):
        return [t]


class TorchComm:
    """torch.distributed collectives (NCCL for CUDA tensors, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_reduce_(self, t):
        self.dist.all_reduce(t, group=self.group)
        return t

    def all_gather(self, t):
        out = [t.new_empty(t.shape) for _ in range(self.world)]
        self.dist.all_gather(out, t.contiguous(), group=self.group)
        return out


def default_comm():
    try:
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
            return TorchComm()
    except ImportError:
        pass
    return LocalComm()


def select_k_smallest(stats, index_base: int, k: int, ops, comm):
    """Global k smallest of the sharded statistics.

    Returns (indices, values, threshold) on every rank: indices ascending
    (int64 tensor), values the matching statistics, threshold the k-th
    smallest statistic (generation.py:159-169)."""
    torch = N.torch_mod()
    st = ops.init(k, stats.device)
    for p in range(8):
        h = ops.hist(stats, st, p)
        comm.all_reduce_(h)
        ops.pick(h, st, p)
    if comm.world == 1:
        quota = ops.k_rem(st)
    else:
        c = ops.counts(stats, st)
        allc = torch.stack(comm.all_gather(c))  # [world, 2]
        eq = allc[:, 1]
        before = eq[: comm.rank].sum() if comm.rank else torch.zeros((), dtype=eq.dtype, device=eq.device)
        quota = torch.clamp(ops.k_rem(st) - before, min=0)
        quota = torch.minimum(quota, eq[comm.rank : comm.rank + 1]).contiguous()
    idx, val, n_out = ops.compact(stats, index_base, st, quota, cap=k)
    thr = ops.threshold(st)
    if comm.world == 1:
        n = int(n_out.item())
        return idx[:n], val[:n], thr
    sizes = torch.stack(comm.all_gather(n_out)).reshape(-1)
    size_list = [int(s) for s in sizes.tolist()]
    mx = max(1, max(size_list))
    pad_i = torch.zeros(mx, dtype=idx.dtype, device=idx.device)
    pad_v = torch.zeros(mx, dtype=val.dtype, device=val.device)
    n_local = size_list[comm.rank]
    pad_i[:n_local] = idx[:n_local]
    pad_v[:n_local] = val[:n_local]
    gi = comm.all_gather(pad_i)
    gv = comm.all_gather(pad_v)
    out_i = torch.cat([g[:s] for g, s in zip(gi, size_list)])
    out_v = torch.cat([g[:s] for g, s in zip(gv, size_list)])
    return out_i, out_v, thr
