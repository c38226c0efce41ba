"""Coarse exact transport on the host (reference: exact.py + _simplex.py).

The coarse Kantorovich LP stays on the host, as BASELINE.json's north star
requires.  It runs the native C++ network simplex in libgridot_b200.so
(``gdt_transport_simplex``), which follows the reference's pivot rules
exactly (_simplex.py:31-361), so supports, flows and duals are bit-identical.
``solve_transport_many`` solves a batch of independent LPs on a host thread
pool without holding the GIL.
"""

from __future__ import annotations

import ctypes
import logging
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import GridotError, IterationLimitError, UnbalancedError

__all__ = ["TransportProblem", "SparseCoupling", "DualPotentials", "build_transport_problem",
           "solve_transport", "solve_transport_many", "OffsetTableCost", "REBALANCE_TOLERANCE",
           "LPBatch", "grid_transport_problem", "hungarian_oracle", "wasserstein_1d"]

logger = logging.getLogger(__name__)

REBALANCE_TOLERANCE = 1e-12


@dataclass(frozen=True, eq=False)
class TransportProblem:
    """Balanced instance on the positive supports (exact.py:46-62)."""

    supply: np.ndarray
    demand: np.ndarray
    cost: np.ndarray
    src_index: np.ndarray
    dst_index: np.ndarray

    @property
    def shape(self) -> tuple:
        return self.cost.shape


@dataclass(frozen=True, eq=False)
class SparseCoupling:
    """(row, col, mass) triples (exact.py:65-87)."""

    row: np.ndarray
    col: np.ndarray
    mass: np.ndarray
    shape: tuple

    def row_marginal(self) -> np.ndarray:
        return np.bincount(self.row, weights=self.mass, minlength=self.shape[0])

    def col_marginal(self) -> np.ndarray:
        return np.bincount(self.col, weights=self.mass, minlength=self.shape[1])

    @property
    def total_mass(self) -> float:
        return float(np.sum(self.mass))

    def to_dense(self) -> np.ndarray:
        out = np.zeros(self.shape)
        out[self.row, self.col] = self.mass
        return out


@dataclass(frozen=True, eq=False)
class DualPotentials:
    """Optimal potentials (f[0] = 0) and min_ij C_ij - f_i - g_j (exact.py:90-100)."""

    f: np.ndarray
    g: np.ndarray
    feasibility_slack: float


class OffsetTableCost:
    """Translation-invariant cost on a full coarse grid, never materialised.

    cost(i, j) = table[x_j - x_i + (cd - 1)] for coarse cells i, j of the grid
    ``cdims`` (flat order axis 0 fastest); ``table`` is the Fortran-flattened
    array over offset vectors with extent 2*cd_a - 1 per axis.  The host
    simplex reads it directly (``gdt_transport_simplex_many``); indexing with
    (rows, cols) arrays returns the same doubles the dense matrix holds.
    """

    def __init__(self, table: np.ndarray, cdims: tuple):
        self.table = np.ascontiguousarray(table, dtype=np.float64).ravel(order="F")
        self.cdims = tuple(int(x) for x in cdims)
        n = int(np.prod(self.cdims))
        self.shape = (n, n)
        self.ext = tuple(2 * c - 1 for c in self.cdims)

    def _index(self, rows, cols):
        xi = np.unravel_index(np.asarray(rows), self.cdims, order="F")
        xj = np.unravel_index(np.asarray(cols), self.cdims, order="F")
        off = tuple(b - a + (c - 1) for a, b, c in zip(xi, xj, self.cdims))
        return np.ravel_multi_index(off, self.ext, order="F")

    def __getitem__(self, key):
        rows, cols = key
        return self.table[self._index(rows, cols)]

    def dense(self) -> np.ndarray:
        n = self.shape[0]
        ids = np.arange(n)
        return self[ids[:, None], ids[None, :]]


def _rebalance(s: np.ndarray, t: np.ndarray) -> None:
    drift = float(s.sum() - t.sum())
    if drift == 0.0:
        return
    if abs(drift) > REBALANCE_TOLERANCE:
        raise UnbalancedError(f"total masses differ by {drift:.3e}, beyond "
                              f"{REBALANCE_TOLERANCE:.0e}")
    if drift > 0:
        t[int(np.argmax(t))] += drift
    else:
        s[int(np.argmax(s))] -= drift


def build_transport_problem(supply, demand, cost) -> TransportProblem:
    """Restrict to positive entries and absorb rounding drift (exact.py:103-136)."""
    supply = np.asarray(supply, dtype=np.float64)
    demand = np.asarray(demand, dtype=np.float64)
    si = np.flatnonzero(supply > 0.0)
    di = np.flatnonzero(demand > 0.0)
    if si.size == 0 or di.size == 0:
        raise GridotError("transport needs nonempty supports on both sides")
    s, t = supply[si].copy(), demand[di].copy()
    _rebalance(s, t)
    full = si.size == cost.shape[0] and di.size == cost.shape[1]
    if isinstance(cost, OffsetTableCost):
        if full:
            return TransportProblem(s, t, cost, si, di)
        cost = cost.dense()
    cost = np.asarray(cost)
    if full:
        sub = np.ascontiguousarray(cost, dtype=np.float64)  # full supports: no gather copy
    else:
        sub = np.ascontiguousarray(cost[np.ix_(si, di)], dtype=np.float64)
    return TransportProblem(s, t, sub, si, di)


def _finish(problem: TransportProblem, status: int, bi, bj, bf, u, v, pivots, slack=True):
    if status == 1:
        raise IterationLimitError(f"pivot cap reached after {pivots} pivots")
    if status != 0:
        raise GridotError(f"simplex failed with status {status}")
    keep = bf > 0.0
    coupling = SparseCoupling(bi[keep].copy(), bj[keep].copy(), bf[keep].copy(), problem.shape)
    value = float(np.sum(bf * problem.cost[bi, bj]))
    if slack:
        dense = problem.cost.dense() if isinstance(problem.cost, OffsetTableCost) else problem.cost
        slack = float(np.min(dense - u[:, None] - v[None, :]))
    else:
        slack = float("nan")
    logger.debug("simplex %dx%d: %d pivots, value %.12g, slack %.3g", problem.shape[0],
                 problem.shape[1], pivots, value, slack)
    return coupling, DualPotentials(u, v, slack), value


def solve_transport(problem: TransportProblem, tol: float = 1e-10,
                    max_pivots: int | None = None):
    """Optimal coupling, duals and value (exact.py:156-189) via the native simplex."""
    if isinstance(problem.cost, OffsetTableCost):
        return solve_transport_many([problem], tol=tol, threads=1)[0] if max_pivots is None \
            else solve_transport(TransportProblem(problem.supply, problem.demand,
                                                  problem.cost.dense(), problem.src_index,
                                                  problem.dst_index), tol, max_pivots)
    ns, nt = problem.shape
    nb = ns + nt - 1
    bi, bj = np.empty(nb, np.int64), np.empty(nb, np.int64)
    bf, u, v = np.empty(nb), np.empty(ns), np.empty(nt)
    piv = ctypes.c_int64(0)
    C = np.ascontiguousarray(problem.cost, dtype=np.float64)
    st = N.lib().gdt_transport_simplex(
        N.ptr(C), N.ptr(problem.supply), N.ptr(problem.demand), ns, nt, 0,
        0 if max_pivots is None else int(max_pivots), float(tol), N.ptr(bi), N.ptr(bj),
        N.ptr(bf), N.ptr(u), N.ptr(v), ctypes.byref(piv))
    if st < 0:
        N.check(st, "gdt_transport_simplex")
    return _finish(problem, st, bi, bj, bf, u, v, int(piv.value))


class LPBatch:
    """A batch of LPs for one native call (``gdt_transport_simplex_many_flags``).

    Jobs may be held back until their cost data exists (``hold`` then
    ``release(q)``, callable from another thread while :meth:`run` blocks in
    native code) and consumed as soon as they finish (``finished(q)``,
    ``result(q)``, ``basis(q)``).  ``warm_from`` / ``warm_basis`` as in
    :func:`solve_transport_many`.
    """

    def __init__(self, problems, tol: float = 1e-10, warm_from=None, warm_basis=None,
                 hold=None):
        self.problems = list(problems)
        count = len(self.problems)
        self.tol = float(tol)
        self._keep = []  # every buffer the native call reads stays alive with the batch

        def addr(a):
            self._keep.append(a)
            return a.ctypes.data

        self.ns = np.array([p.shape[0] for p in self.problems], np.int64)
        self.nt = np.array([p.shape[1] for p in self.problems], np.int64)
        self.out = [(np.empty(a + b - 1, np.int64), np.empty(a + b - 1, np.int64),
                     np.empty(a + b - 1), np.empty(a), np.empty(b))
                    for a, b in zip(self.ns, self.nt)]
        ptr = lambda xs: np.array([addr(x) for x in xs], np.uint64)  # noqa: E731
        self.C = np.zeros(count, np.uint64)
        self.T = np.zeros(count, np.uint64)
        self.gnd = np.zeros(count, np.int32)
        self.gdims = np.ones((count, 4), np.int64)
        for q, prob in enumerate(self.problems):
            if isinstance(prob.cost, OffsetTableCost):
                self.T[q] = addr(prob.cost.table)
                self.gnd[q] = len(prob.cost.cdims)
                self.gdims[q, :self.gnd[q]] = prob.cost.cdims
            else:
                cost = prob.cost
                if not (isinstance(cost, np.ndarray) and cost.dtype == np.float64
                        and cost.flags.c_contiguous):
                    cost = np.ascontiguousarray(cost, dtype=np.float64)
                self.C[q] = addr(cost)
        self.sup = ptr([np.ascontiguousarray(p.supply) for p in self.problems])
        self.dem = ptr([np.ascontiguousarray(p.demand) for p in self.problems])
        self.bi, self.bj, self.bf, self.u, self.v = (ptr([o[i] for o in self.out])
                                                     for i in range(5))
        self.wf = (np.full(count, -1, np.int64) if warm_from is None
                   else np.array(warm_from, np.int64))
        if warm_basis is not None:
            for q, wb in enumerate(warm_basis):
                if wb is None:
                    continue
                if self.wf[q] >= 0 or len(wb[0]) != len(self.out[q][0]):
                    raise ValueError("warm_basis: one start per problem, sized ns + nt - 1")
                for dst, src in zip(self.out[q][:3], wb):
                    dst[:] = src
                self.wf[q] = q
        self.ready = np.ones(count, np.int32)
        if hold is not None:
            self.ready[np.asarray(hold, dtype=np.int64)] = 0
        self.done = np.zeros(count, np.int32)
        self.status = np.full(count, -999, np.int32)
        self.pivots = np.zeros(count, np.int64)

    def release(self, q) -> None:
        """Let held job(s) q start (their cost data is now in place)."""
        self.ready[q] = 1

    def run(self, threads: int = 0) -> None:
        if len(self.problems) == 0:
            return
        N.check(N.lib().gdt_transport_simplex_many_flags(
            len(self.problems), N.ptr(self.C), N.ptr(self.T), N.ptr(self.gnd),
            N.ptr(self.gdims), N.ptr(self.sup), N.ptr(self.dem), N.ptr(self.ns), N.ptr(self.nt),
            N.ptr(self.wf), self.tol, N.ptr(self.bi), N.ptr(self.bj), N.ptr(self.bf),
            N.ptr(self.u), N.ptr(self.v), N.ptr(self.status), N.ptr(self.pivots), int(threads),
            N.ptr(self.ready), N.ptr(self.done)), "gdt_transport_simplex_many_flags")

    def finished(self, q) -> bool:
        return bool(self.done[q])

    def result(self, q, slack: bool = False):
        """(coupling, duals, value) of job q, or the exception it raised."""
        st = int(self.status[q])
        try:
            if st < 0:
                raise GridotError(f"simplex failed with native status {st}")
            return _finish(self.problems[q], st, *self.out[q], int(self.pivots[q]), slack=slack)
        except GridotError as exc:
            return exc

    def value(self, q):
        """Optimal value of job q only (no coupling / duals), or its exception."""
        st = int(self.status[q])
        if st == 1:
            return IterationLimitError(f"pivot cap reached after {int(self.pivots[q])} pivots")
        if st != 0:
            return GridotError(f"simplex failed with status {st}")
        bi, bj, bf = self.out[q][:3]
        return float(np.sum(bf * self.problems[q].cost[bi, bj]))

    def basis(self, q):
        """Final basis (bi, bj, bf) of job q, None if it failed."""
        return self.out[q][:3] if int(self.status[q]) in (0,) else None


def solve_transport_many(problems, tol: float = 1e-10, threads: int = 0, warm_from=None,
                         slack: bool = True, warm_basis=None, return_basis: bool = False):
    """Solve a batch of problems on `threads` host threads (0 = all cores).

    ``warm_from[q] = w`` (w < q, same supports and marginals) starts problem q
    from the optimal basis of problem w instead of the northwest corner;
    ``warm_basis[q] = (bi, bj, bf)`` (a feasible spanning-tree basis of q's
    marginals, e.g. the final basis of an earlier solve on the same supports)
    starts it from that basis.  The optimal value is unchanged (the LP optimum
    is unique), only the pivot path differs.  Problems without a warm start
    follow the reference's pivot sequence exactly.  Returns a list of
    (coupling, duals, value) or the exception each raised -- and, with
    ``return_basis``, also the list of final bases (bi, bj, bf) (None where the
    solve failed); ``slack=False`` skips the O(ns*nt) feasibility diagnostic
    of DualPotentials.
    """
    count = len(problems)
    if count == 0:
        return ([], []) if return_basis else []
    batch = LPBatch(problems, tol=tol, warm_from=warm_from, warm_basis=warm_basis)
    batch.run(threads)
    res = [batch.result(q, slack=slack) for q in range(count)]
    if return_basis:
        return res, [None if isinstance(r, Exception) else batch.out[q][:3]
                     for q, r in enumerate(res)]
    return res


# ---------------------------------------------------------------------------
# fine-grid instances and the validation oracles (exact.py:139-153, 197-253)
# ---------------------------------------------------------------------------


def grid_transport_problem(mu, nu, p: float, metric: str = "l2") -> TransportProblem:
    """Fine-scale instance between two grid measures under rho^p costs
    (exact.py:139-153): supports, rebalanced masses, dense support cost."""
    from .costs import pairwise_costs

    if metric != "l2":
        raise ValueError(f"unsupported metric {metric!r}")
    mu_idx, nu_idx = mu.support, nu.support
    if mu_idx.size == 0 or nu_idx.size == 0:
        raise GridotError("transport needs nonempty supports on both sides")
    sup, dem = mu.mass[mu_idx].copy(), nu.mass[nu_idx].copy()
    _rebalance(sup, dem)
    cost = pairwise_costs(mu.grid.coordinates()[mu_idx], nu.grid.coordinates()[nu_idx], p)
    return TransportProblem(sup, dem, np.ascontiguousarray(cost), mu_idx, nu_idx)


def hungarian_oracle(problem: TransportProblem, denom: int) -> float:
    """Exact value by unit splitting and an assignment solve (exact.py:197-224);
    every mass must be a multiple of 1/denom.  Small instances only."""
    from scipy.optimize import linear_sum_assignment

    from .errors import QuantizationResidualError

    ks_f, kd_f = problem.supply * denom, problem.demand * denom
    res = max(float(np.abs(ks_f - np.round(ks_f)).max()), float(np.abs(kd_f - np.round(kd_f)).max()))
    if res > 1e-9:
        raise QuantizationResidualError(f"masses are not multiples of 1/{denom} "
                                        f"(residual {res:.3e})")
    ks, kd = np.round(ks_f).astype(np.int64), np.round(kd_f).astype(np.int64)
    if ks.sum() != kd.sum():
        raise UnbalancedError(f"unit counts differ: {int(ks.sum())} vs {int(kd.sum())}")
    cost = problem.cost.dense() if isinstance(problem.cost, OffsetTableCost) else problem.cost
    unit = np.asarray(cost)[np.ix_(np.repeat(np.arange(ks.size), ks),
                                   np.repeat(np.arange(kd.size), kd))]
    rows, cols = linear_sum_assignment(unit)
    return float(unit[rows, cols].sum()) / denom


def wasserstein_1d(mu, nu, p: float) -> float:
    """Closed-form W_p on a 1-D grid (exact.py:227-253): |F_mu - F_nu| summed
    for p = 1, quantile slivers swept in lockstep otherwise."""
    from .errors import DimensionMismatchError, GridMismatchError

    if mu.grid.ndim != 1 or nu.grid.ndim != 1:
        raise DimensionMismatchError("wasserstein_1d needs 1-dimensional grids")
    if mu.grid != nu.grid:
        raise GridMismatchError(f"grids differ: {mu.grid.dims} vs {nu.grid.dims}")
    if abs(mu.total_mass - nu.total_mass) > 1e-9:
        raise UnbalancedError(f"total masses differ: {mu.total_mass!r} vs {nu.total_mass!r}")
    cm, cn = np.cumsum(mu.mass), np.cumsum(nu.mass)
    if p == 1.0:
        return float(np.sum(np.abs(cm - cn)))
    n = mu.grid.cell_count
    pos = np.arange(1, n + 1, dtype=np.float64)
    levels = np.union1d(cm, cn)
    dq = np.diff(np.concatenate(([0.0], levels)))
    iu = np.minimum(np.searchsorted(cm, levels, side="left"), n - 1)
    iv = np.minimum(np.searchsorted(cn, levels, side="left"), n - 1)
    return float(np.sum(dq * np.abs(pos[iu] - pos[iv]) ** p)) ** (1.0 / p)
