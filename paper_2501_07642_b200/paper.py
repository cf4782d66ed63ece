"""The paper's entry point names (arXiv 2501.07642 Sec. 6)
mapped onto the fastrr-compatible engine."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .generation import DesignSpec, RandomizationPool, generate_pool, pool_assignment_matrix
from .keys import MASK64


@dataclass
class Randomizations(RandomizationPool):
    """Result of :func:`generate_randomizations`: a pool that also answers to
    the paper's field names (``randomizations``, ``balance``)."""

    @property
    def randomizations(self) -> np.ndarray:
        return pool_assignment_matrix(self)

    @property
    def balance(self) -> np.ndarray:
        return self.stats


def generate_randomizations(n_units: int, n_treated: int, X, randomization_type: str = "monte_carlo",
                            randomization_accept_prob: float = 0.01, max_draws: int = 100_000,
                            batch_size: int = 10_000, approximate_inv: bool = False, file=None,
                            seed: int | None = None, storage: str = "keys", verbose: bool = False,
                            enumeration_cap: int | None = None) -> Randomizations:
    """Pool of acceptable randomizations, exact or Monte Carlo.

    ``approximate_inv=True`` selects the ridge-regularised inverse (the
    paper's high-dimensional option); ``file`` streams the accepted pool to
    a CSV; ``seed`` is the 64-bit root seed of the candidate keys."""
    kw = {}
    if enumeration_cap is not None:
        kw["enumeration_cap"] = int(enumeration_cap)
    design = DesignSpec(
        n_units=int(n_units), n_treated=int(n_treated), accept_prob=float(randomization_accept_prob),
        mode=randomization_type, max_draws=int(max_draws),
        batch_size=int(min(batch_size, max_draws)) if randomization_type == "monte_carlo" else int(batch_size),
        precision_mode="ridge" if approximate_inv else "exact", root_seed=int(seed or 0) & MASK64,
        storage=storage, **kw)
    pool = generate_pool(X, design, out_path=file)
    out = Randomizations(**{f: getattr(pool, f) for f in ("design", "stats", "threshold_value", "n_candidates",
                                                          "accepted_indices", "keys", "assignments")})
    if verbose:
        print(f"accepted {out.n_accepted} of {out.n_candidates} candidate randomizations "
              f"(threshold {out.threshold_value:.6g})")
    return out
