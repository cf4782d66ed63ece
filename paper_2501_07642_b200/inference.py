"""Randomization tests over an accepted pool (drop-in for fastrr inference.py).

The pool's statistics are computed on the GPU straight from keys (the
assignment is regenerated in shared memory and never materialised) or from
explicit assignment rows: difference in means of Y with numpy's pairwise
reduction order, the same for Y = W_obs (exact popcounts), and pool
membership of W_obs.  p(tau) = #{|a - tau b| >= |tau_obs - tau b_obs|} / M
is an integer count over the pool, evaluated for whole tau grids (and whole
bisection trees) per launch.  The fiducial-interval control flow is the
reference's (inference.py:185-250), so results are bit-identical.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass, replace

import numpy as np

from . import _native as N
from . import keys as keymod
from ._select import default_comm
from .errors import (
    DimensionError,
    EmptyIntervalError,
    EmptyPoolError,
    InvalidDesignError,
    UnsupportedStatisticError,
)
from .generation import DesignSpec, RandomizationPool, pool_assignment_matrix
from .keys import Assignment

_BISECT_DEPTH = 6  # bisection levels evaluated per launch (2^6 - 1 taus)


@dataclass
class TestResult:
    """Outcome of a randomization test (inference.py:41-54)."""

    __test__ = False  # not a pytest class

    p_value: float
    tau_obs: float
    fi: tuple[float, float] | None
    stat_distribution: np.ndarray
    alpha: float | None = None
    obs_in_pool: bool = True

    @property
    def n_accepted(self) -> int:
        return int(self.stat_distribution.shape[0])


def _as_vector(x, name: str) -> np.ndarray:
    v = np.asarray(x.bits if isinstance(x, Assignment) else x)
    if v.ndim != 1:
        raise DimensionError(f"{name} must be one-dimensional, got shape {v.shape}")
    return v


def _check_lengths(w: np.ndarray, y: np.ndarray):
    if w.shape[0] != y.shape[0]:
        raise DimensionError(f"assignment length {w.shape[0]} does not match outcome length {y.shape[0]}")


def diff_in_means(W, Y) -> float:
    """mean(Y | W=1) - mean(Y | W=0) for one assignment (inference.py:71-79)."""
    w = _as_vector(W, "assignment")
    y = np.asarray(Y, dtype=np.float64)
    _check_lengths(w, y)
    t = int(w.sum())
    if not (0 < t < w.shape[0]):
        raise InvalidDesignError("assignment must treat at least one and leave one control")
    return float(y[w == 1].mean() - y[w == 0].mean())


def _resolve_statistic(statistic):
    if statistic is None or statistic is diff_in_means or statistic == "diff_in_means":
        return None
    if callable(statistic):
        return statistic
    raise UnsupportedStatisticError(f"unknown statistic {statistic!r}")


# ------------------------------------------------------------- device side
def _pack_bits(w: np.ndarray) -> np.ndarray:
    """uint32 words, bit e of word e // 32 = unit e treated (frr.h layout)."""
    n = w.shape[0]
    words = (n + 31) // 32
    padded = np.zeros(words * 32, dtype=np.uint8)
    padded[:n] = w != 0
    return np.packbits(padded, bitorder="little").view("<u4").astype(np.uint32)


class _PoolStats:
    """Device a, b (+ membership) of a pool for outcome y and observed w.

    Under torch.distributed (world > 1) every rank computes a and b for its
    contiguous shard of the pool only; the integer counts of p(tau) are
    all-reduced (SURVEY section 8 e), and the full a -- needed only for
    stat_distribution and np.std in the fiducial interval -- is gathered in
    rank order on first use."""

    def __init__(self, pool: RandomizationPool, obs_w: np.ndarray, y: np.ndarray):
        torch = N.torch_mod()
        dev = N.device()
        d = pool.design
        n, t = d.n_units, d.n_treated
        self.m = pool.n_accepted
        y_dev = torch.from_numpy(np.ascontiguousarray(y, dtype=np.float64)).to(dev)
        obs_dev = torch.from_numpy(_pack_bits(obs_w).view(np.int32)).to(dev)
        match = torch.zeros(1, dtype=torch.int32, device=dev)
        self.comm = comm = default_comm()
        lo, hi = self.m * comm.rank // comm.world, self.m * (comm.rank + 1) // comm.world
        a = torch.empty(hi - lo, dtype=torch.float64, device=dev)
        b = torch.empty(hi - lo, dtype=torch.float64, device=dev)
        if pool.assignments is not None:
            rows_dev = torch.from_numpy(np.ascontiguousarray(pool.assignments[lo:hi], dtype=np.int8)).to(dev)
            if hi > lo:
                N.call("frr_dim_rows", N.ptr(rows_dev), hi - lo, n, t, N.ptr(y_dev), N.ptr(obs_dev), N.ptr(a),
                       N.ptr(b), N.ptr(match), N.stream_ptr())
        else:
            if pool.keys is None:
                # the reference's pool_assignment_matrix -> regenerate_assignments
                # raises this for a pool without keys (generation.py:349-352)
                raise InvalidDesignError(
                    "pool stores no keys; exact-mode pools carry explicit assignments instead")
            if hi > lo:
                self._dim_keys(pool.keys[lo:hi], int(d.root_seed) & keymod.MASK64, n, t, y_dev, obs_dev, a, b,
                               match)
        if comm.world > 1:
            comm.all_reduce_(match)
        self.a_local, self.b_local = a, b
        self._a_full = a if comm.world == 1 else None
        self.in_pool = bool(int(match.sum().item()) != 0)
        # observed statistic through the same reduction (inference.py:124, 174-177)
        t_obs = int(obs_w.sum())
        obs_row = torch.from_numpy(np.ascontiguousarray(obs_w, dtype=np.int8).reshape(1, -1)).to(dev)
        ab = torch.empty(2, dtype=torch.float64, device=dev)
        N.call("frr_dim_rows", N.ptr(obs_row), 1, n, t_obs, N.ptr(y_dev), N.ptr(obs_dev), N.ptr(ab[0:1]),
               N.ptr(ab[1:2]), None, N.stream_ptr())
        tau_obs, b_obs = ab.cpu().tolist()
        self.tau_obs, self.b_obs = float(tau_obs), float(b_obs)

    @staticmethod
    def _dim_keys(keys, root_seed, n, t, y_dev, obs_dev, a, b, match):
        """frr_dim_mc_ws over the keys [m, 2] (host), chunk by chunk: the
        upload of chunk i + 1 runs on a side stream under the statistics of
        chunk i (the library's own chunks, so launch shapes do not change)."""
        torch = N.torch_mod()
        dev = a.device
        m = int(keys.shape[0])
        keys = np.ascontiguousarray(keys, dtype=np.uint64).view(np.int64)
        ws_bytes = int(N.lib().frr_dim_mc_workspace_bytes(m, n))
        ws = torch.empty(max(1, ws_bytes), dtype=torch.uint8, device=dev)
        chunk = max(1, int(N.lib().frr_dim_mc_chunk_keys(m, n, t, ws_bytes)))
        main = torch.cuda.current_stream(dev)
        side = torch.cuda.Stream(dev)
        side.wait_stream(main)

        def upload(lo):
            with torch.cuda.stream(side):
                kd = torch.from_numpy(keys[lo:lo + chunk]).to(dev, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(side)
            return kd, ev

        nxt = upload(0)
        for lo in range(0, m, chunk):
            kd, ev = nxt
            main.wait_event(ev)
            kd.record_stream(main)
            draws = kd[:, 1].contiguous()
            N.call("frr_dim_mc_ws", root_seed, N.ptr(draws), int(kd.shape[0]), n, t, N.ptr(y_dev), N.ptr(obs_dev),
                   N.ptr(a[lo:]), N.ptr(b[lo:]), N.ptr(match), N.ptr(ws), ws_bytes, N.stream_ptr())
            if lo + chunk < m:
                nxt = upload(lo + chunk)  # (a pageable upload blocks the host while chunk lo computes)

    @property
    def a(self):
        """The whole pool's a in pool order (gathered across ranks once)."""
        if self._a_full is None:
            self._a_full = self._gather(self.comm, self.a_local)
        return self._a_full

    @staticmethod
    def _gather(comm, a):
        torch = N.torch_mod()
        n_local = torch.tensor([a.shape[0]], dtype=torch.int64, device=a.device)
        sizes = [int(s) for s in torch.stack(comm.all_gather(n_local)).reshape(-1).tolist()]
        mx = max(1, max(sizes))
        pa = torch.zeros(mx, dtype=a.dtype, device=a.device)
        pa[: a.shape[0]] = a
        ga = comm.all_gather(pa)
        return torch.cat([g[:s] for g, s in zip(ga, sizes)])

    def counts(self, taus, rhs) -> np.ndarray:
        """#{|a - tau b| >= rhs} over the whole pool for each (tau, rhs) pair:
        one launch on this rank's shard, then an int64 all-reduce."""
        torch = N.torch_mod()
        taus = np.ascontiguousarray(taus, dtype=np.float64)
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        dev = self.a_local.device
        tt = torch.from_numpy(np.concatenate([taus, rhs])).to(dev)
        out = torch.zeros(taus.shape[0], dtype=torch.int64, device=dev)
        m_local = int(self.a_local.shape[0])
        if m_local:
            N.call("frr_tau_counts", N.ptr(self.a_local), N.ptr(self.b_local), m_local,
                   N.ptr(tt[: taus.shape[0]]), N.ptr(tt[taus.shape[0]:]), taus.shape[0], N.ptr(out),
                   N.stream_ptr())
        if self.comm.world > 1:
            self.comm.all_reduce_(out)
        return out.cpu().numpy()


def randomization_pvalue(obs_w, obs_y, pool: RandomizationPool, statistic=None) -> TestResult:
    """Two-sided randomization test against the accepted pool (inference.py:129-159)."""
    w = _as_vector(obs_w, "observed assignment").astype(np.int8)
    y = np.asarray(obs_y, dtype=np.float64)
    _check_lengths(w, y)
    if not np.isfinite(y).all():
        raise InvalidDesignError("outcomes contain non-finite entries")
    if w.shape[0] != pool.design.n_units:
        raise DimensionError(
            f"observed assignment has {w.shape[0]} units but pool was built for {pool.design.n_units}")
    custom = _resolve_statistic(statistic)
    if pool.n_accepted == 0:
        raise EmptyPoolError("pool has no accepted randomizations")
    if custom is not None:
        # user-supplied Python statistic: evaluated on the host over the
        # GPU-regenerated rows (not part of the accelerated path)
        mat = pool_assignment_matrix(pool)
        dist = np.array([custom(row, y) for row in mat], dtype=np.float64)
        tau_obs = float(custom(w, y))
        in_pool = bool((mat == w).all(axis=1).any())
    else:
        ps = _PoolStats(pool, w, y)
        dist = N.to_host(ps.a)
        tau_obs = ps.tau_obs
        in_pool = ps.in_pool
    if not in_pool:
        warnings.warn("observed assignment is not a member of the accepted pool; "
                      "the p-value may fall below 1/n_accepted", stacklevel=2)
    if custom is None:
        count = int(ps.counts([0.0], [abs(tau_obs)])[0])
    else:
        count = int(np.count_nonzero(np.abs(dist) >= abs(tau_obs)))
    return TestResult(p_value=float(count) / dist.shape[0], tau_obs=tau_obs, fi=None,
                      stat_distribution=dist, alpha=None, obs_in_pool=in_pool)


def fiducial_interval(obs_w, obs_y, pool: RandomizationPool, alpha: float = 0.05,
                      statistic=None) -> tuple[float, float]:
    """Additive effects not rejected at level alpha (inference.py:185-250)."""
    if _resolve_statistic(statistic) is not None:
        raise UnsupportedStatisticError("fiducial intervals support only the difference-in-means statistic")
    if not (0.0 < alpha < 1.0):
        raise InvalidDesignError(f"alpha must lie in (0, 1), got {alpha}")
    w = _as_vector(obs_w, "observed assignment").astype(np.int8)
    y = np.asarray(obs_y, dtype=np.float64)
    _check_lengths(w, y)
    if pool.n_accepted == 0:
        raise EmptyPoolError("pool has no accepted randomizations")
    ps = _PoolStats(pool, w, y)
    return _fi_from_stats(ps, alpha)


def _fi_from_stats(ps: _PoolStats, alpha: float, a_host=None) -> tuple[float, float]:
    """a_host: the pool's a already on the host (else it is copied here)."""
    tau_obs, b_obs, m = ps.tau_obs, ps.b_obs, ps.m

    def p_many(taus) -> np.ndarray:
        taus = list(taus)
        rhs = [abs(tau_obs - tau * b_obs) for tau in taus]
        return ps.counts(taus, rhs).astype(np.float64) / m

    half = 10.0 * float(np.std(N.to_host(ps.a) if a_host is None else a_host))
    if not np.isfinite(half) or half == 0.0:
        half = max(1.0, abs(tau_obs))
    lo_g, hi_g = tau_obs - half, tau_obs + half
    for _ in range(64):
        grid = np.linspace(lo_g, hi_g, 201)
        pvals = p_many(grid)
        accept = pvals >= alpha
        if not accept.any():
            raise EmptyIntervalError(
                f"no effect size reaches p >= {alpha}; maximum p on the grid is {float(pvals.max())}",
                max_p=float(pvals.max()))
        if accept[0] or accept[-1]:
            width = hi_g - lo_g
            lo_g, hi_g = lo_g - width, hi_g + width
            continue
        break
    else:
        raise EmptyIntervalError("acceptance region did not close under grid expansion; alpha may be "
                                 "below the 1/n_accepted resolution of the pool")
    tol = 1e-6 * max(1.0, abs(tau_obs))
    first = int(np.argmax(accept))
    last = len(accept) - 1 - int(np.argmax(accept[::-1]))

    def refine(outside: float, inside: float) -> float:
        # the reference's sequential bisection, evaluated _BISECT_DEPTH levels
        # per launch: every node of the next levels' decision tree is a
        # deterministic function of (inside, outside), so the walk below
        # visits exactly the midpoints the sequential loop would.
        while abs(inside - outside) > tol:
            nodes = []

            def expand(o, i, depth):
                if depth == 0 or not abs(i - o) > tol:
                    return
                mid = 0.5 * (i + o)
                nodes.append(mid)
                expand(o, mid, depth - 1)   # accepted: inside = mid
                expand(mid, i, depth - 1)   # rejected: outside = mid

            expand(outside, inside, _BISECT_DEPTH)
            pv = dict(zip(nodes, p_many(nodes)))
            for _ in range(_BISECT_DEPTH):
                if not abs(inside - outside) > tol:
                    break
                mid = 0.5 * (inside + outside)
                if pv[mid] >= alpha:
                    inside = mid
                else:
                    outside = mid
        return inside

    lower = refine(float(grid[first - 1]), float(grid[first]))
    upper = refine(float(grid[last + 1]), float(grid[last]))
    return (float(lower), float(upper))


def randomization_test(obs_w=None, obs_y=None, pool: RandomizationPool | None = None, statistic=None,
                       find_fi: bool = False, alpha: float = 0.05, *, obsW=None, obsY=None,
                       candidate_randomizations=None, findFI=None, test_statistic=None) -> TestResult:
    """p-value plus optional fiducial interval (inference.py:253-266).

    Also accepts the paper's argument names: ``obsW``,
    ``obsY``, ``candidate_randomizations`` (a pool or an r x n 0/1 matrix),
    ``findFI`` and ``test_statistic``."""
    if obsW is not None:
        obs_w = obsW
    if obsY is not None:
        obs_y = obsY
    if findFI is not None:
        find_fi = bool(findFI)
    if test_statistic is not None:
        statistic = test_statistic
    if candidate_randomizations is not None:
        pool = candidate_randomizations
    if obs_w is None or obs_y is None or pool is None:
        raise InvalidDesignError("randomization_test needs obs_w, obs_y and a pool")
    if not isinstance(pool, RandomizationPool):
        pool = _pool_from_matrix(np.asarray(pool))
    if statistic is None or _resolve_statistic(statistic) is None:
        # one device pass serves both the p-value and the interval
        w = _as_vector(obs_w, "observed assignment").astype(np.int8)
        y = np.asarray(obs_y, dtype=np.float64)
        _check_lengths(w, y)
        if not np.isfinite(y).all():
            raise InvalidDesignError("outcomes contain non-finite entries")
        if w.shape[0] != pool.design.n_units:
            raise DimensionError(
                f"observed assignment has {w.shape[0]} units but pool was built for {pool.design.n_units}")
        if pool.n_accepted == 0:
            raise EmptyPoolError("pool has no accepted randomizations")
        if find_fi and not (0.0 < alpha < 1.0):
            raise InvalidDesignError(f"alpha must lie in (0, 1), got {alpha}")
        ps = _PoolStats(pool, w, y)
        if not ps.in_pool:
            warnings.warn("observed assignment is not a member of the accepted pool; "
                          "the p-value may fall below 1/n_accepted", stacklevel=2)
        count = int(ps.counts([0.0], [abs(ps.tau_obs)])[0])
        res = TestResult(p_value=float(count) / ps.m, tau_obs=ps.tau_obs, fi=None,
                         stat_distribution=N.to_host(ps.a), alpha=None, obs_in_pool=ps.in_pool)
        if find_fi:
            res.fi = _fi_from_stats(ps, alpha, res.stat_distribution)
            res.alpha = alpha
        return res
    res = randomization_pvalue(obs_w, obs_y, pool, statistic=statistic)
    if find_fi:
        res.fi = fiducial_interval(obs_w, obs_y, pool, alpha=alpha, statistic=statistic)
        res.alpha = alpha
    return res


def _pool_from_matrix(mat: np.ndarray) -> RandomizationPool:
    mat = np.ascontiguousarray(mat, dtype=np.int8)
    if mat.ndim != 2 or mat.shape[0] == 0:
        raise DimensionError("candidate_randomizations must be a nonempty r x n matrix")
    t = int(mat[0].sum())
    if not (mat.sum(axis=1) == t).all():
        raise InvalidDesignError("candidate randomizations must share one treated count")
    design = DesignSpec(n_units=mat.shape[1], n_treated=t, accept_prob=1.0, mode="exact")
    return RandomizationPool(design=design, stats=np.zeros(mat.shape[0]), threshold_value=0.0,
                             n_candidates=mat.shape[0], accepted_indices=np.arange(mat.shape[0]),
                             assignments=mat)


def _observed_from_rule(rule, pool: RandomizationPool) -> np.ndarray:
    if isinstance(rule, str):
        if rule != "first":
            raise InvalidDesignError(f"unknown observed-assignment rule {rule!r}")
        return pool_assignment_matrix(pool)[0]
    if callable(rule):
        return np.asarray(rule(pool), dtype=np.int8)
    return _as_vector(rule, "observed assignment").astype(np.int8)


def threshold_sweep(X, base_design: DesignSpec, probs, obs_y, obs_w_rule="first", find_fi: bool = False,
                    alpha: float = 0.05, workers: int | None = None) -> list[dict]:
    """Pool + test per acceptance probability, same seed and draw count
    (inference.py:279-312); failing rows are recorded and the sweep goes on.

    Candidate statistics do not depend on the acceptance probability, so
    pass 1 (generation + balance check) runs once on the GPU and every row
    only re-runs the exact selection -- the pools equal the reference's
    per-row rebuilds."""
    from .generation import _Pass1, _resolve_workers

    rows = []
    p1, p1_error = None, None
    try:
        _resolve_workers(workers)
        p1 = _Pass1(X, base_design)
    except Exception as exc:  # every row would fail the same way
        p1_error = exc
    for prob in probs:
        row = {"accept_prob": float(prob), "p_value": None, "n_accepted": None, "status": "ok"}
        if find_fi:
            row["fi_width"] = None
        try:
            design = replace(base_design, accept_prob=float(prob))
            if p1_error is not None:
                raise p1_error
            pool = p1.pool(design)
            res = randomization_test(_observed_from_rule(obs_w_rule, pool), obs_y, pool, find_fi=find_fi,
                                     alpha=alpha)
            row["p_value"] = res.p_value
            row["n_accepted"] = res.n_accepted
            if find_fi and res.fi is not None:
                row["fi_width"] = res.fi[1] - res.fi[0]
        except Exception as exc:  # row-level isolation
            row["status"] = f"failed: {exc}"
        rows.append(row)
    return rows
