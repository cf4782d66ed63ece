"""Synthetic experiments: the simulation config, the keyed polar-method
normal stream, ``simulate_data`` and the accelerator cost model
(reference bench.py:43-154).

These produce *inputs* for the hot path (covariates, outcomes, the observed
assignment).  The keyed streams and the polar-method candidate pairs are
computed on the GPU (frr_sim_pairs: splitmix64 outputs, uniforms and
s = v1^2 + v2^2 in the reference's exact arithmetic); the accepted pairs'
scale sqrt(-2 ln s / s) is numpy's, so the normals are bit-identical to the
reference's on the same machine (its logarithm is numpy's).  The observed
assignment is regenerated from its key on the GPU like any other
candidate.  The reference's timing harness (``run_benchmark`` /
``summarize_benchmark``, which times its own naive/batched/parallel CPU
paths) is out of scope: this package's measurement is ``bench.py``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import keys as keymod
from .balance import CovariateMatrix
from .errors import InvalidDesignError

SIM_STREAM_BASE = 1 << 63  # simulation draw indices never collide with candidate draws


@dataclass(frozen=True)
class SimConfig:
    """Shape and outcome model of one synthetic experiment (bench.py:43-67)."""

    n: int
    k: int
    max_draws: int = 10_000
    batch_size: int = 10_000
    tau_true: float = 1.0
    noise_sd: float = 0.5
    coef: np.ndarray | None = None
    replicates: int = 10

    def __post_init__(self):
        if self.n < 4 or self.n % 2:
            raise InvalidDesignError(f"n must be an even count >= 4, got {self.n}")
        if self.k < 1:
            raise InvalidDesignError(f"k must be positive, got {self.k}")
        if self.replicates < 1:
            raise InvalidDesignError("replicates must be at least 1")
        if self.coef is not None:
            c = np.asarray(self.coef, dtype=np.float64)
            if c.shape != (self.k,):
                raise InvalidDesignError(f"coef must have length k={self.k}")
            object.__setattr__(self, "coef", c)


@dataclass(frozen=True)
class CostModel:
    """Batched balance-check runtime model (bench.py:70-92): per-draw cost
    k = alpha * d, fixed costs r_cpu / r_gpu, accelerator throughput beta."""

    r_cpu: float
    r_gpu: float
    alpha: float
    d: int
    beta: float
    M: int
    B: int = 1

    def __post_init__(self):
        for name in ("r_cpu", "r_gpu", "alpha", "beta", "M", "B", "d"):
            if getattr(self, name) < 0:
                raise InvalidDesignError(f"{name} must be nonnegative")
        if self.beta < 1:
            raise InvalidDesignError("beta must be at least 1")


def estimate_speedup(model: CostModel) -> float:
    """Predicted (r_cpu + k M) / (r_gpu + k M / beta) (bench.py:89-98)."""
    work = model.alpha * model.d * model.M
    denom = model.r_gpu + work / model.beta
    if denom <= 0:
        raise InvalidDesignError("cost model denominator must be positive")
    return (model.r_cpu + work) / denom


def _polar_pairs(seed: int, stream: int, pair_lo: int, npairs: int):
    """(v1, v2, s) of polar-method pairs [pair_lo, pair_lo + npairs) of a
    simulation stream, on the GPU (frr_sim_pairs), returned to the host."""
    from . import _native as N

    torch = N.torch_mod()
    out = torch.empty((3, npairs), dtype=torch.float64, device=N.device())
    N.call("frr_sim_pairs", N.ctypes.c_uint64(int(seed) & keymod.MASK64), N.ctypes.c_uint64(int(stream)), pair_lo,
           npairs, N.ptr(out[0]), N.ptr(out[1]), N.ptr(out[2]), N.stream_ptr())
    h = out.cpu().numpy()
    return h[0], h[1], h[2]


def normals_from_stream(seed: int, stream: int, count: int) -> np.ndarray:
    """Standard normals by the polar method on a keyed stream (bench.py:107-136).

    Outputs 2j, 2j+1 form pair j: uniforms v = 2 (u >> 11) 2^-53 - 1, kept
    when 0 < s = v1^2 + v2^2 < 1, giving (v1, v2) sqrt(-2 ln s / s); kept
    pairs are consumed in order, so the values do not depend on chunking."""
    out = np.empty(count, dtype=np.float64)
    filled, pair = 0, 0
    while filled < count:
        want = (count - filled + 1) // 2
        take = max(64, int(1.3 * want) + 16)  # ~21% of pairs are rejected
        v1, v2, s = _polar_pairs(seed, stream, pair, take)
        ok = (s > 0.0) & (s < 1.0)
        g = np.sqrt(-2.0 * np.log(s[ok]) / s[ok])
        z = np.empty(2 * int(ok.sum()), dtype=np.float64)
        z[0::2] = v1[ok] * g
        z[1::2] = v2[ok] * g
        room = min(z.shape[0], count - filled)
        out[filled:filled + room] = z[:room]
        filled += room
        pair += take
    return out


def simulate_data(cfg: SimConfig, seed: int = 0):
    """(CovariateMatrix, observed Assignment, outcomes) of one synthetic
    experiment (bench.py:139-154): streams 0 covariates (row-major),
    1 coefficients (unless cfg.coef), 2 noise; the assignment is the key
    (seed, 2^63 + 3) with n/2 treated."""
    X = normals_from_stream(seed, 0, cfg.n * cfg.k).reshape(cfg.n, cfg.k)
    coef = cfg.coef if cfg.coef is not None else normals_from_stream(seed, 1, cfg.k)
    noise = normals_from_stream(seed, 2, cfg.n)
    obs = keymod.assignment_from_key(keymod.AssignmentKey(seed, SIM_STREAM_BASE + 3), cfg.n, cfg.n // 2)
    y = X @ coef + cfg.tau_true * obs.bits + cfg.noise_sd * noise
    return CovariateMatrix(X), obs, y
