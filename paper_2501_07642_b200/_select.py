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

import math
import os

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
        """Order-preserving compaction; at most `cap` entries are written,
        n_out holds the full count."""
        torch = self.torch
        m = int(stats.shape[0])
        cap = max(1, min(int(cap), m))
        idx = torch.empty(cap, dtype=torch.int64, device=st.device)
        val = torch.empty(cap, dtype=torch.float64, device=st.device)
        n_out = torch.empty(1, dtype=torch.int64, device=st.device)
        ws = torch.empty(int(N.lib().frr_select_workspace_bytes(m)) // 8 + 1, dtype=torch.int64, device=st.device)
        N.call("frr_select_compact_capped", N.ptr(stats), m, int(index_base), N.ptr(st), N.ptr(quota), cap,
               N.ptr(idx), N.ptr(val), N.ptr(n_out), N.ptr(ws), N.stream_ptr())
        return idx, val, n_out

    # (fill_ with a Python scalar is a device fill; `st[1] = -1` would be a
    # blocking host-to-device copy that waits for everything queued before it)
    def set_threshold(self, st, bits: int):
        """State whose threshold is the given bit pattern (all 64 bits fixed)."""
        st[0:1].fill_(int(np.array([bits], dtype=np.uint64).view(np.int64)[0]))
        st[1:2].fill_(-1)

    def set_threshold_from(self, st, src):
        """set_threshold with the bit pattern of src's threshold, on the device."""
        st[0:1].copy_(src[0:1])
        st[1:2].fill_(-1)

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
    """torch.distributed collectives: NCCL for CUDA tensors (the GPU path).

    Under a gloo group (no CUDA collectives) CUDA tensors are staged through
    host memory -- e.g. several ranks sharing one GPU for testing, or a
    debugging run without NCCL; the results are the same, only slower."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.stage = dist.get_backend(group) == "gloo"

    def all_reduce_(self, t):
        if self.stage and t.is_cuda:
            h = t.cpu()
            self.dist.all_reduce(h, group=self.group)
            t.copy_(h)
            return t
        self.dist.all_reduce(t, group=self.group)
        return t

    def all_gather(self, t):
        if self.stage and t.is_cuda:
            h = t.contiguous().cpu()
            out = [h.new_empty(h.shape) for _ in range(self.world)]
            self.dist.all_gather(out, h, group=self.group)
            return [o.to(t.device) for o in out]
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


# debug hook (tools / bench FRR_BENCH_DEBUG): (label, perf_counter) marks
TRACE = None
FALLBACKS = 0  # narrowed selects that fell back to the full data (diagnostics)


def _mark(label):
    if TRACE is not None:
        import time

        TRACE.append((label, time.perf_counter()))


SAMPLE = 1 << 20          # statistics sampled to bound the threshold from above
PREFILTER_MIN = 1 << 22   # global candidate count from which the narrowing pays
PREFILTER_MAX_Q = 0.05    # acceptance fractions above this select on the full data


def _upper_bound_bits(stats, k: int, m_total: int, ops, comm):
    """Bit pattern h of a statistic that bounds the k-th smallest from above
    with overwhelming probability: the k_s-th smallest of a strided sample
    (same on every rank), k_s = q s + 8 sqrt(q s) + 16 for q = k / M.  A bad
    bound is detected by the caller (fewer than k statistics <= h) and only
    costs a fall back to the full select."""
    m = int(stats.shape[0])
    s_r = sample_size(m, comm)
    stride = max(1, m // s_r)
    return bound_from_sample(stats[::stride][:s_r].contiguous(), k, m_total, ops, comm)


def sample_size(m: int, comm) -> int:
    """Per-rank sample length (equal on every rank for shards >= SAMPLE)."""
    return max(1, min(m, SAMPLE // comm.world))


def bound_from_sample(sample, k: int, m_total: int, ops, comm):
    """(h, fraction) of _upper_bound_bits from this rank's sample of
    sample_size(m) statistics; the samples of all ranks are gathered so that
    every rank gets the same h."""
    torch = N.torch_mod()
    s_r = sample_size(int(sample.shape[0]), comm) if comm.world == 1 else SAMPLE // comm.world
    if sample.shape[0] < s_r:  # keep shapes equal across ranks
        sample = torch.cat([sample, sample.new_full((s_r - sample.shape[0],), float("inf"))])
    if comm.world > 1:
        sample = torch.cat(comm.all_gather(sample))
    st, frac = _bound_state(sample, k, m_total, ops)
    _mark("bound launched")
    h = int(st[0].item()) & ((1 << 64) - 1)
    _mark("bound read")
    return h, frac


def _bound_state(sample, k: int, m_total: int, ops):
    """Select state whose threshold (st[0]) is the bound h of the gathered
    sample, left on the device; and the sampled fraction k_s / s."""
    s = int(sample.shape[0])
    qs = k / m_total * s
    k_s = min(s, int(math.ceil(qs + 8.0 * math.sqrt(qs) + 16)))
    st = ops.init(k_s, sample.device)
    for p in range(8):
        ops.pick(ops.hist(sample, st, p), st, p)
    return st, k_s / s


def select_k_smallest(stats, index_base: int, k: int, ops, comm, prefilter: bool = True, m_total=None):
    """Global k smallest of the sharded statistics.

    Returns (indices, values, threshold) on every rank: indices ascending
    (int64 tensor), values the matching statistics, threshold the k-th
    smallest statistic (generation.py:159-169).

    For large inputs the select first narrows to C = {i: stat_i <= h} (one
    ordered compaction pass; h an upper bound of the threshold from a
    sample), then runs the radix passes and the final compaction on C: two
    passes over the full statistics instead of ten.  Every statistic <= the
    threshold is in C, so the result is the same as on the full data."""
    return select_start(stats, index_base, k, ops, comm, prefilter, m_total).finish()


class SelectJob:
    """A select whose kernels are all enqueued; finish() reads the result
    back (the only host synchronisation) and, if the narrowing failed, runs
    the select on the full statistics.  The statistics must stay unchanged
    until finish() returns."""

    def __init__(self, finish):
        self._finish = finish

    def finish(self):
        return self._finish()


def select_start(stats, index_base: int, k: int, ops, comm, prefilter: bool = True, m_total=None) -> SelectJob:
    """Enqueue the select of select_k_smallest without waiting for it
    (m_total: the global statistics count when the caller knows it, which
    saves a collective and its host read)."""
    torch = N.torch_mod()
    if m_total is None:
        m_total = int(stats.shape[0])
        if comm.world > 1:
            mt = torch.tensor([m_total], dtype=torch.int64, device=stats.device)
            m_total = int(comm.all_reduce_(mt).item())
    if os.environ.get("FRR_SELECT_PREFILTER") == "0":  # A/B knob
        prefilter = False
    if prefilter and m_total >= PREFILTER_MIN and k <= PREFILTER_MAX_Q * m_total:
        # Every kernel of the narrowed select is enqueued without a host
        # round trip (the bound, the narrowed count and the tie quota stay
        # on the device), so a host thread that stalls while they run costs
        # no GPU time: the narrowed buffer's unused tail holds +inf, which
        # never enters a selection of k <= count finite statistics.  The
        # two ways the narrowing can fail -- a capped buffer that overflowed
        # or fewer than k statistics under the bound -- are checked once at
        # the end and fall back to the select on the full data.
        m = int(stats.shape[0])
        s_r = sample_size(m, comm)
        sample = stats[:: max(1, m // s_r)][:s_r].contiguous()
        if comm.world > 1:
            r_s = SAMPLE // comm.world
            if sample.shape[0] < r_s:  # keep shapes equal across ranks
                sample = torch.cat([sample, sample.new_full((r_s - sample.shape[0],), float("inf"))])
            sample = torch.cat(comm.all_gather(sample))
        st_h, qh = _bound_state(sample, k, m_total, ops)
        sth = ops.init(k, stats.device)
        ops.set_threshold_from(sth, st_h)
        everything = torch.full((1,), (1 << 63) - 1, dtype=torch.int64, device=stats.device)
        cap = int(qh * m * 1.25) + 4096
        c_idx, c_val, c_n = ops.compact(stats, index_base, sth, everything, cap)
        _mark("compact launched")
        pos = torch.arange(c_val.shape[0], device=c_val.device)
        c_val = c_val.masked_fill(pos >= c_n, float("inf"))
        over = (c_n > c_val.shape[0]).to(torch.int64)
        tot = c_n.clone()
        if comm.world > 1:
            comm.all_reduce_(over)
            comm.all_reduce_(tot)
        job = _full_start(c_val, 0, k, ops, comm, idx_map=c_idx)
        rb = _Readback.of(job, over, tot)

        def finish():
            if rb is not None:
                n, bits, ov, tt, sizes = rb.values()
            else:
                n, bits, ov, tt, sizes = None, None, int(over.item()), int(tot.item()), None
            if ov == 0 and tt >= k:
                res = _full_finish(job, comm, n, bits, sizes)
                _mark("narrowed ok")
                return res
            global FALLBACKS
            FALLBACKS += 1
            return _full_finish(_full_start(stats, index_base, k, ops, comm), comm)

        return SelectJob(finish)
    job = _full_start(stats, index_base, k, ops, comm)
    rb = _Readback.of(job)
    if rb is None:
        return SelectJob(lambda: _full_finish(job, comm))

    def finish_full():
        n, bits, sizes = rb.values()
        return _full_finish(job, comm, n, bits, sizes)

    return SelectJob(finish_full)


class _Readback:
    """The select's result scalars -- this rank's count, the threshold bits,
    for the narrowing its overflow flag and total, and under several ranks
    every rank's count -- copied to page-locked host memory in stream order
    right behind the select's kernels and collectives, with an event: a
    later finish() waits for that event only, not for work enqueued after
    the select (the bench keeps later passes queued behind it)."""

    SLOTS = 64  # read-backs alive at once (the bench keeps 4 selects in flight)
    WIDTH = 4 + 256  # scalars + up to 256 ranks' counts
    _ring = None
    _next = 0

    def __init__(self, scalars, sizes=None):
        torch = N.torch_mod()
        cls = type(self)
        if cls._ring is None:
            # one page-locked block for all slots, allocated once: a fresh
            # page-locked allocation (cudaHostAlloc) can stall the host for
            # tens of ms, which must not happen while a pipeline is running
            cls._ring = torch.empty((cls.SLOTS, cls.WIDTH), dtype=torch.int64, pin_memory=True)
        n_sizes = 0 if sizes is None else int(sizes.shape[0])
        self.n_scalars = len(scalars)
        self.host = cls._ring[cls._next % cls.SLOTS, : len(scalars) + n_sizes]
        cls._next += 1
        for i, t in enumerate(scalars):
            self.host[i : i + 1].copy_(t.reshape(-1)[:1], non_blocking=True)
        if n_sizes:
            self.host[len(scalars):].copy_(sizes.reshape(-1), non_blocking=True)
        self.has_sizes = sizes is not None
        self.ev = torch.cuda.Event()
        self.ev.record()

    @classmethod
    def of(cls, job, *extra):
        idx, val, n_out, st, ops, idx_map, gathered = job
        if not n_out.is_cuda:
            return None
        sizes = gathered[0] if gathered is not None else None
        if sizes is not None and (not sizes.is_cuda or sizes.shape[0] > cls.WIDTH - 4):
            return None
        return cls([n_out, st[0:1], *extra], sizes)

    def values(self):
        """[scalars..., sizes list or None]"""
        self.ev.synchronize()
        v = [int(x) for x in self.host.tolist()]
        return v[: self.n_scalars] + [v[self.n_scalars:] if self.has_sizes else None]


def _select_full(stats, index_base: int, k: int, ops, comm, idx_map=None):
    """The radix select proper; idx_map (narrowed input) maps local positions
    to global indices before the gather."""
    return _full_finish(_full_start(stats, index_base, k, ops, comm, idx_map), comm)


def _full_start(stats, index_base: int, k: int, ops, comm, idx_map=None):
    """Enqueue the radix passes and the final compaction (no host read)."""
    torch = N.torch_mod()
    st = ops.init(k, stats.device)
    _mark("full init")
    for p in range(8):
        h = ops.hist(stats, st, p)
        comm.all_reduce_(h)
        ops.pick(h, st, p)
    _mark("full hist")
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
    if idx_map is not None:
        # map to global indices now, in stream order (entries past the count
        # are unwritten: clamped into range, sliced off at the read-back)
        idx = idx_map[idx.clamp(0, max(0, idx_map.shape[0] - 1))]
        idx_map = None
    gathered = None
    if comm.world > 1:
        # the rank-ordered gather, enqueued now with buffers of the maximum
        # count k (every rank's count is <= k): the host learns the counts
        # only at the read-back
        sizes = torch.cat(comm.all_gather(n_out.reshape(1)))
        pad_i = torch.zeros(k, dtype=idx.dtype, device=idx.device)
        pad_v = torch.zeros(k, dtype=val.dtype, device=val.device)
        pad_i[: idx.shape[0]] = idx[:k]
        pad_v[: val.shape[0]] = val[:k]
        gathered = (sizes, comm.all_gather(pad_i), comm.all_gather(pad_v))
    _mark("final launched")
    return idx, val, n_out, st, ops, idx_map, gathered


def _full_finish(job, comm, n=None, bits=None, sizes=None):
    """Read back the select enqueued by _full_start: (indices, values,
    threshold); n, bits and sizes: this rank's count, the threshold bits and
    every rank's count when a _Readback already has them."""
    torch = N.torch_mod()
    idx, val, n_out, st, ops, idx_map, gathered = job
    if bits is None:
        thr = ops.threshold(st)
    else:
        thr = float(np.array([bits & ((1 << 64) - 1)], dtype=np.uint64).view(np.float64)[0])
    _mark("final read")
    if comm.world == 1:
        if n is None:
            n = int(n_out.item())
        return idx[:n], val[:n], thr
    size_t, gi, gv = gathered
    size_list = [int(x) for x in (sizes if sizes is not None else size_t.tolist())]
    out_i = torch.cat([g[:c] for g, c in zip(gi, size_list)])
    out_v = torch.cat([g[:c] for g, c in zip(gv, size_list)])
    return out_i, out_v, thr
