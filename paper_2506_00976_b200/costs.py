"""Ground costs and the three coarse cost matrices (reference: costs.py).

* C-tilde (block centres) and C-min (closed-form nearest-point gap) depend only
  on (grid, kappa, p); they are computed once per configuration on the host
   and cached.
* C-bar (marginally weighted block average, costs.py:128-171) is the
  O(N^{2d}) stage and runs in libgridot_b200.so (kernel K2): exact mode
  reproduces the reference's rounding order bit for bit; fast mode (fp32
  precision of BASELINE.json) uses block moments for p = 2 and fp32 tiles
  otherwise.
* ``cost_table`` tabulates rho^p over the integer squared distances of a grid
  with numpy's own ``sq ** (p/2)`` so the device reads bit-identical costs for
  any p.
"""

from __future__ import annotations

import functools
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .device import device, stream, to_dev, to_host, torch
from .errors import DimensionMismatchError, GridMismatchError
from .measures import CoarseningSpec, GridMeasure, GridSpec, coarsen_grid, pad_batch

__all__ = ["CostSpec", "CoarseCostMatrix", "pairwise_costs", "ground_cost",
           "center_cost_matrix", "weighted_cost_matrix", "min_cost_matrix", "cost_table",
           "weighted_cost_batch"]


def _sq_dists(xa: np.ndarray, xb: np.ndarray) -> np.ndarray:
    out = np.zeros((xa.shape[0], xb.shape[0]))
    for a in range(xa.shape[1]):
        diff = xa[:, a][:, None] - xb[:, a][None, :]
        out += diff * diff
    return out


def _power(sq, p: float):
    if p == 2.0:
        return sq
    if p == 1.0:
        return np.sqrt(sq)
    return sq ** (p / 2.0)


def pairwise_costs(xa: np.ndarray, xb: np.ndarray, p: float, metric: str = "l2") -> np.ndarray:
    """rho(xa_i, xb_j)^p for small host blocks (costs.py:44-53)."""
    if metric != "l2":
        raise ValueError(f"unsupported metric {metric!r}")
    return _power(_sq_dists(np.asarray(xa, float), np.asarray(xb, float)), p)


@dataclass(frozen=True, eq=False)
class CostSpec:
    """Lazy rho^p cost between two point clouds (costs.py:56-99)."""

    source: np.ndarray
    target: np.ndarray
    p: float
    metric: str = "l2"

    def __post_init__(self):
        s = np.ascontiguousarray(self.source, dtype=np.float64)
        t = np.ascontiguousarray(self.target, dtype=np.float64)
        if s.ndim != 2 or t.ndim != 2 or s.shape[1] != t.shape[1]:
            raise DimensionMismatchError(
                f"coordinate arrays must be (n, d) with matching d, got {s.shape} and {t.shape}")
        if self.metric != "l2":
            raise ValueError(f"unsupported metric {self.metric!r}")
        if not self.p >= 1.0:
            raise ValueError(f"p must be >= 1, got {self.p}")
        object.__setattr__(self, "source", s)
        object.__setattr__(self, "target", t)
        object.__setattr__(self, "p", float(self.p))

    @property
    def n_source(self) -> int:
        return self.source.shape[0]

    @property
    def n_target(self) -> int:
        return self.target.shape[0]

    def block(self, rows, cols) -> np.ndarray:
        return pairwise_costs(self.source[rows], self.target[cols], self.p)

    def full(self) -> np.ndarray:
        return pairwise_costs(self.source, self.target, self.p)


def ground_cost(spec: CostSpec, i: int, j: int) -> float:
    d = spec.source[i] - spec.target[j]
    return float(np.dot(d, d) ** (spec.p / 2.0))


@dataclass(frozen=True, eq=False)
class CoarseCostMatrix:
    """Dense coarse cost matrix; ``unused`` flags filler entries (costs.py:108-118)."""

    kind: str
    values: np.ndarray
    unused: np.ndarray | None = None


@functools.lru_cache(maxsize=64)
def cost_table(max_sq: int, p: float) -> np.ndarray:
    """rho^p for every integer squared distance 0..max_sq (numpy's power)."""
    return np.ascontiguousarray(_power(np.arange(max_sq + 1, dtype=np.float64), float(p)))


def max_sq_of(dims) -> int:
    return int(sum((n - 1) * (n - 1) for n in dims))


def center_cost_matrix(src_centers: np.ndarray, dst_centers: np.ndarray,
                       p: float) -> CoarseCostMatrix:
    return CoarseCostMatrix("center", pairwise_costs(src_centers, dst_centers, p))


@functools.lru_cache(maxsize=32)
def centre_cost_cached(dims: tuple, kappa: int, p: float) -> np.ndarray:
    c = coarsen_grid(GridSpec(dims), CoarseningSpec(kappa))
    out = pairwise_costs(c, c, p)
    out.setflags(write=False)
    return out


@functools.lru_cache(maxsize=32)
def min_cost_cached(dims: tuple, kappa: int, p: float) -> np.ndarray:
    """Closed-form per-axis gap max(0, kappa|k-l| - (kappa-1)) (costs.py:174-192)."""
    cd = CoarseningSpec(kappa).coarse_dims(GridSpec(dims))
    pos = np.column_stack(np.unravel_index(np.arange(int(np.prod(cd))), cd, order="F"))
    pos = pos.astype(np.float64)
    sq = np.zeros((pos.shape[0], pos.shape[0]))
    for a in range(len(cd)):
        gap = np.maximum(kappa * np.abs(pos[:, a][:, None] - pos[:, a][None, :]) - (kappa - 1), 0.0)
        sq += gap * gap
    out = sq ** (p / 2.0)
    out.setflags(write=False)
    return out


def _offset_grid(cdims):
    """Offset vectors D (per axis -(cd-1)..cd-1), Fortran-flattened: [count, d]."""
    ext = tuple(2 * c - 1 for c in cdims)
    axes = np.unravel_index(np.arange(int(np.prod(ext))), ext, order="F")
    return np.column_stack([a - (c - 1) for a, c in zip(axes, cdims)]).astype(np.float64)


@functools.lru_cache(maxsize=32)
def centre_cost_table(dims: tuple, kappa: int, p: float):
    """C-tilde as an offset table: same doubles as centre_cost_cached (kappa*D)."""
    from .exact import OffsetTableCost

    cd = CoarseningSpec(kappa).coarse_dims(GridSpec(dims))
    D = _offset_grid(cd) * kappa
    sq = np.zeros(D.shape[0])
    for a in range(D.shape[1]):
        sq += D[:, a] * D[:, a]
    return OffsetTableCost(_power(sq, float(p)), cd)


@functools.lru_cache(maxsize=32)
def min_cost_table(dims: tuple, kappa: int, p: float):
    """C-min as an offset table: same doubles as min_cost_cached."""
    from .exact import OffsetTableCost

    cd = CoarseningSpec(kappa).coarse_dims(GridSpec(dims))
    D = _offset_grid(cd)
    sq = np.zeros(D.shape[0])
    for a in range(D.shape[1]):
        gap = np.maximum(kappa * np.abs(D[:, a]) - (kappa - 1), 0.0)
        sq += gap * gap
    return OffsetTableCost(sq ** (p / 2.0), cd)


def min_cost_matrix(grid: GridSpec, coarsening: CoarseningSpec, p: float) -> CoarseCostMatrix:
    return CoarseCostMatrix("min", min_cost_cached(grid.dims, coarsening.kappa, float(p)).copy())


def weighted_cost_batch(mu_pad, nu_pad, mu_c, nu_c, padded_dims, kappa, p, mode, ctil_dev=None,
                        table_dev=None, want_unused=True):
    """Device C-bar for a batch: returns (values [B,n,n] f64, unused [B,n,n] u8
    or None when ``want_unused`` is False -- the kernels then skip the mask)."""
    t = torch()
    B = mu_pad.shape[0]
    n = mu_c.shape[1]
    if ctil_dev is None:
        ctil_dev = to_dev(centre_cost_cached(tuple(padded_dims), kappa, float(p)))
    ms = max_sq_of(padded_dims)
    if table_dev is None and p not in (1.0, 2.0):
        table_dev = to_dev(cost_table(ms, float(p)))
    ops = N.torch_ops()
    if ops is not None and not want_unused:  # the PyTorch extension's operator
        out = ops.weighted_cost(mu_pad, nu_pad, mu_c, nu_c, ctil_dev, table_dev, int(ms),
                                [int(d) for d in padded_dims], int(kappa), float(p), int(mode))
        return out, None
    out = t.empty((B, n, n), dtype=t.float64, device=mu_pad.device)
    unused = t.empty((B, n, n), dtype=t.uint8, device=mu_pad.device) if want_unused else None
    N.check(N.lib().gdt_weighted_cost(
        N.ptr(mu_pad), N.ptr(nu_pad), N.ptr(mu_c), N.ptr(nu_c), N.ptr(ctil_dev), N.ptr(table_dev),
        ms, N.ptr(out), N.ptr(unused), B, len(padded_dims), N.i64s(padded_dims), kappa, float(p),
        int(mode), stream()), "gdt_weighted_cost")
    return out, unused


def weighted_cost_matrix(mu: GridMeasure, nu: GridMeasure, coarsening: CoarseningSpec,
                         p: float) -> CoarseCostMatrix:
    """C-bar on the device, bit-exact with the reference (costs.py:128-171)."""
    if mu.grid != nu.grid:
        raise GridMismatchError(f"grids differ: {mu.grid.dims} vs {nu.grid.dims}")
    from .measures import sumpool_batch

    device()
    k = coarsening.kappa
    x = to_dev(np.stack([mu.mass, nu.mass]))
    xp, pd = pad_batch(x, mu.grid.dims, k)
    sums = sumpool_batch(x, mu.grid.dims, k)
    vals, unused = weighted_cost_batch(xp[0:1], xp[1:2], sums[0:1], sums[1:2], pd, k, float(p),
                                       0)
    return CoarseCostMatrix("weighted", to_host(vals)[0], to_host(unused)[0].astype(bool))
