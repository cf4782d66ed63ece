"""Key-addressed treatment assignments (drop-in for fastrr keys.py).

The key -> assignment contract is the reference's to the bit
(keys.py:9-38): state = mix64((seed ^ draw*C) + C), stream
u_j = mix64(state + j*C), rejection-sampled bounds, partial Fisher-Yates.
The scalar key helpers (``mix64``, ``derive_state``) are plain integer
functions of the wire contract; every assignment is generated on the GPU
by libfrr (``frr_regen_mc``), including the single-key path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import InvalidDesignError

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB
KEY_WORDS = 2


@dataclass(frozen=True)
class AssignmentKey:
    """Two-word handle (root seed, draw index) of one candidate (keys.py:58-78)."""

    root_seed: int
    draw_index: int

    def __post_init__(self):
        for name in ("root_seed", "draw_index"):
            v = getattr(self, name)
            if not (0 <= int(v) <= MASK64):
                raise InvalidDesignError(f"{name} must be an unsigned 64-bit integer, got {v!r}")

    def to_bytes(self) -> bytes:
        return int(self.root_seed).to_bytes(8, "little") + int(self.draw_index).to_bytes(8, "little")

    @classmethod
    def from_bytes(cls, raw: bytes) -> "AssignmentKey":
        if len(raw) != 16:
            raise InvalidDesignError(f"serialized key must be 16 bytes, got {len(raw)}")
        return cls(int.from_bytes(raw[:8], "little"), int.from_bytes(raw[8:], "little"))


@dataclass(frozen=True)
class Assignment:
    """A 0/1 treatment vector with its treated count (keys.py:81-96)."""

    bits: np.ndarray
    n_treated: int

    def __post_init__(self):
        b = np.ascontiguousarray(self.bits, dtype=np.int8)
        b.setflags(write=False)
        object.__setattr__(self, "bits", b)
        if int(b.sum()) != self.n_treated:
            raise InvalidDesignError("assignment bits do not sum to n_treated")

    @property
    def n_units(self) -> int:
        return self.bits.shape[0]


def mix64(z: int) -> int:
    """splitmix64 finaliser on a Python int (keys.py:99-104)."""
    z &= MASK64
    z = ((z ^ (z >> 30)) * _M1) & MASK64
    z = ((z ^ (z >> 27)) * _M2) & MASK64
    return z ^ (z >> 31)


def derive_state(key: AssignmentKey) -> int:
    """Generator state of a key (keys.py:118-121)."""
    return mix64(((key.root_seed ^ ((key.draw_index * GOLDEN) & MASK64)) + GOLDEN) & MASK64)


def _check_design(n_units: int, n_treated: int):
    if n_units < 2:
        raise InvalidDesignError(f"n_units must be at least 2, got {n_units}")
    if not (0 < n_treated < n_units):
        raise InvalidDesignError(
            f"n_treated must satisfy 0 < n_treated < n_units, got n_treated={n_treated}, n_units={n_units}")


def _as_draws(draw_indices) -> np.ndarray:
    draws = np.asarray(draw_indices)
    if draws.dtype != np.uint64:
        if draws.size and int(draws.min()) < 0:
            raise InvalidDesignError("draw indices must be nonnegative")
        draws = draws.astype(np.uint64)
    return np.ascontiguousarray(draws.reshape(-1))


def to_device_u64(a: np.ndarray):
    """Upload a uint64 array (as the int64 bit pattern) to the current GPU."""
    torch = N.torch_mod()
    dev = N.device()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint64).view(np.int64)).to(dev)


def regen_rows_device(root_seed: int, draws_dev, n_units: int, n_treated: int):
    """int8 [m, n] device tensor of the assignments of keys (root_seed, draws)."""
    torch = N.torch_mod()
    m = int(draws_dev.shape[0])
    rows = torch.empty((m, n_units), dtype=torch.int8, device=draws_dev.device)
    N.call("frr_regen_mc", int(root_seed) & MASK64, N.ptr(draws_dev), m, n_units, n_treated,
           N.ptr(rows), None, N.stream_ptr())
    return rows


def regen_bits_device(root_seed: int, draws_dev, n_units: int, n_treated: int):
    """Packed uint32 [m, ceil(n/32)] device tensor (bit e = unit e treated)."""
    torch = N.torch_mod()
    m = int(draws_dev.shape[0])
    words = (n_units + 31) // 32
    bits = torch.empty((m, words), dtype=torch.int32, device=draws_dev.device)
    N.call("frr_regen_mc", int(root_seed) & MASK64, N.ptr(draws_dev), m, n_units, n_treated,
           None, N.ptr(bits), N.stream_ptr())
    return bits


def batch_assignments(root_seed: int, draw_indices, n_units: int, n_treated: int) -> np.ndarray:
    """int8 ``len(draw_indices) x n_units`` matrix, row i the assignment of
    key (root_seed, draw_indices[i]) -- keys.py:177-208, on the GPU."""
    _check_design(n_units, n_treated)
    draws = _as_draws(draw_indices)
    if draws.shape[0] == 0:
        return np.zeros((0, n_units), dtype=np.int8)
    rows = regen_rows_device(root_seed, to_device_u64(draws), n_units, n_treated)
    return N.to_host(rows)


def assignment_from_key(key: AssignmentKey, n_units: int, n_treated: int) -> Assignment:
    """Regenerate the assignment addressed by ``key`` (keys.py:138-159)."""
    _check_design(n_units, n_treated)
    row = batch_assignments(key.root_seed, np.array([key.draw_index], dtype=np.uint64), n_units, n_treated)[0]
    return Assignment(bits=row, n_treated=n_treated)


def memory_improvement_factor(n_units: int, key_words: int = KEY_WORDS) -> float:
    """Storage ratio of full vectors to keys, n / L (keys.py:211-215)."""
    if key_words < 1:
        raise InvalidDesignError(f"key_words must be at least 1, got {key_words}")
    return n_units / key_words
