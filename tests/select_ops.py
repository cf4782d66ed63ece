"""Test-side restatement of the libfrr select kernels in numpy (the checker
ops that let the multi-rank orchestration run over gloo on CPU)."""

import numpy as np
import torch


class NumpySelectOps:
    def init(self, k, device):
        return torch.tensor([0, 0, k, 0], dtype=torch.int64)

    def _bits(self, stats):
        return stats.numpy().view(np.uint64)

    def hist(self, stats, st, p):
        b = self._bits(stats)
        prefix, mask = np.uint64(int(st[0]) & (2**64 - 1)), np.uint64(int(st[1]) & (2**64 - 1))
        sel = b[(b & mask) == prefix]
        digits = ((sel >> np.uint64(56 - 8 * p)) & np.uint64(255)).astype(np.int64)
        return torch.from_numpy(np.bincount(digits, minlength=256).astype(np.int64))

    def pick(self, hist, st, p):
        k = int(st[2])
        cum = np.cumsum(hist.numpy())
        digit = int(np.searchsorted(cum, k))
        before = int(cum[digit - 1]) if digit else 0
        prefix = (int(st[0]) & (2**64 - 1)) | (digit << (56 - 8 * p))
        mask = (int(st[1]) & (2**64 - 1)) | (255 << (56 - 8 * p))
        st[0] = np.array([prefix], dtype=np.uint64).view(np.int64)[0]
        st[1] = np.array([mask], dtype=np.uint64).view(np.int64)[0]
        st[2] = k - before

    def counts(self, stats, st):
        b = self._bits(stats)
        T = np.uint64(int(st[0]) & (2**64 - 1))
        return torch.tensor([int((b < T).sum()), int((b == T).sum())], dtype=torch.int64)

    def k_rem(self, st):
        return st[2:3]

    def compact(self, stats, index_base, st, quota, cap):
        b = self._bits(stats)
        T = np.uint64(int(st[0]) & (2**64 - 1))
        q = int(quota.reshape(-1)[0])
        eq_idx = np.flatnonzero(b == T)[: max(q, 0)]
        idx = np.sort(np.concatenate([np.flatnonzero(b < T), eq_idx]))
        return (torch.from_numpy(idx + index_base), stats[torch.from_numpy(idx)],
                torch.tensor([idx.shape[0]], dtype=torch.int64))

    def set_threshold(self, st, bits):
        st[0] = int(np.array([bits], dtype=np.uint64).view(np.int64)[0])
        st[1] = -1

    def set_threshold_from(self, st, src):
        st[0] = src[0]
        st[1] = -1

    def threshold(self, st):
        return float(np.array([int(st[0]) & (2**64 - 1)], dtype=np.uint64).view(np.float64)[0])
