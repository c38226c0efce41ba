"""The four quantization bounds and their building blocks (reference: quantized.py).

Same names, signatures and report contracts as the reference
(quantized.py:172, 199, 288, 487); every call routes through the batched
device engine (engine.py) with a batch of one pair.  ``precision`` is an
addition: "fp64" (default) reproduces the reference's arithmetic order,
"fp32" is the fast mode of BASELINE.json (bounds within 1e-5 relative).

Building blocks kept for API parity: ``UpscaleKernel``, ``upscale_coupling``
(host materialisation of the fine triples -- the bound itself never
materialises them), ``interpolate_potential`` and ``c_transform`` (device).
"""

from __future__ import annotations

import itertools
import logging
import time
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import _native as N
from .costs import CostSpec
from .device import device, stream, to_dev, to_host, torch
from .engine import quantized_bounds
from .errors import DimensionMismatchError, GridMismatchError
from .exact import SparseCoupling
from .measures import GridMeasure, GridSpec

__all__ = ["UpscaleKernel", "upscale_coupling", "weighted_cost_upper_bound",
           "min_cost_lower_bound", "primal_upscaling_upper_bound", "interpolate_potential",
           "c_transform", "dual_upscaling_lower_bound"]

logger = logging.getLogger(__name__)


@dataclass(frozen=True, eq=False)
class UpscaleKernel:
    """Normalised (kappa,)*2d spreading weights (quantized.py:57-103)."""

    kappa: int
    ndim: int
    weights: np.ndarray

    def __post_init__(self):
        if self.kappa < 1:
            raise ValueError(f"kappa must be >= 1, got {self.kappa}")
        if self.ndim < 1:
            raise ValueError(f"ndim must be >= 1, got {self.ndim}")
        w = np.ascontiguousarray(self.weights, dtype=np.float64)
        want = (self.kappa,) * (2 * self.ndim)
        if w.shape != want:
            raise DimensionMismatchError(f"kernel weights must have shape {want}, got {w.shape}")
        if (w < 0.0).any() or not np.isfinite(w).all():
            raise ValueError("kernel weights must be finite and nonnegative")
        total = float(w.sum())
        if total <= 0.0:
            raise ValueError("kernel weights must have positive total")
        object.__setattr__(self, "weights", w / total)

    @classmethod
    def uniform(cls, kappa: int, ndim: int) -> "UpscaleKernel":
        cells = kappa ** (2 * ndim)
        return cls(kappa, ndim, np.full((kappa,) * (2 * ndim), 1.0 / cells))

    def paired(self) -> np.ndarray:
        """(kappa^d, kappa^d): row = source offset, col = target offset."""
        m = self.kappa ** self.ndim
        return self.weights.reshape((m, m), order="F")


def _block_cells(ids, cdims, fdims, kappa) -> np.ndarray:
    d = len(cdims)
    off = np.column_stack(np.unravel_index(np.arange(kappa ** d), (kappa,) * d, order="F"))
    blk = np.column_stack(np.unravel_index(np.asarray(ids), cdims, order="F"))
    fine = blk[:, None, :] * kappa + off[None, :, :]
    return np.ravel_multi_index(tuple(fine[..., a] for a in range(d)), fdims, order="F")


def upscale_coupling(coarse: SparseCoupling, kernel: UpscaleKernel,
                     fine_dims: tuple) -> SparseCoupling:
    """Explicit fine triples (cell_t(k), cell_s(l), m*W[t,s]) (quantized.py:119-159)."""
    k, d = kernel.kappa, kernel.ndim
    fine_dims = tuple(int(x) for x in fine_dims)
    if len(fine_dims) != d:
        raise DimensionMismatchError(f"fine dims {fine_dims} do not match kernel dimension {d}")
    if any(n % k for n in fine_dims):
        raise DimensionMismatchError(f"fine dims {fine_dims} are not multiples of kappa={k}")
    cdims = tuple(n // k for n in fine_dims)
    nc = int(np.prod(cdims))
    if coarse.shape != (nc, nc):
        raise DimensionMismatchError(
            f"coupling shape {coarse.shape} does not match coarse grid {cdims}")
    R = _block_cells(coarse.row, cdims, fine_dims, k)
    C = _block_cells(coarse.col, cdims, fine_dims, k)
    mass = np.asarray(coarse.mass)[:, None, None] * kernel.paired()[None, :, :]
    rows = np.broadcast_to(R[:, :, None], mass.shape).ravel()
    cols = np.broadcast_to(C[:, None, :], mass.shape).ravel()
    mass = mass.ravel()
    keep = mass > 0.0
    nf = int(np.prod(fine_dims))
    return SparseCoupling(rows[keep], cols[keep], mass[keep], (nf, nf))


def _one_ring_spread_host(rows, cols, mass, cdims, fdims, kappa):
    """3^d-ring respread, duplicates summed (quantized.py:250-285); cold path."""
    d = len(cdims)
    shifts = np.array(list(itertools.product((-1, 0, 1), repeat=d)))
    lim = np.array(cdims)

    def ring(fid):
        base = np.array(np.unravel_index(int(fid), cdims, order="F"))
        cand = base[None, :] + shifts
        cand = cand[np.all((cand >= 0) & (cand < lim[None, :]), axis=1)]
        return np.ravel_multi_index(tuple(cand[:, a] for a in range(d)), cdims, order="F")

    R, C, M = [], [], []
    for r, c, m in zip(rows, cols, mass):
        rc = _block_cells(ring(r), cdims, fdims, kappa).ravel()
        cc = _block_cells(ring(c), cdims, fdims, kappa).ravel()
        rr, c2 = np.meshgrid(rc, cc, indexing="ij")
        R.append(rr.ravel())
        C.append(c2.ravel())
        M.append(np.full(rr.size, m / (rc.size * cc.size)))
    n = int(np.prod(fdims))
    mat = sp.coo_array((np.concatenate(M), (np.concatenate(R), np.concatenate(C))),
                       shape=(n, n))
    mat.sum_duplicates()
    logger.warning("upscaled support cannot reach a positive marginal; "
                   "respreading over one coarse ring")
    return mat.coords[0].astype(np.int64), mat.coords[1].astype(np.int64), mat.data


def _same_grid(mu: GridMeasure, nu: GridMeasure) -> None:
    if mu.grid != nu.grid:
        raise GridMismatchError(f"grids differ: {mu.grid.dims} vs {nu.grid.dims}")


def _one(mu, nu, kappa, p, method, **kw):
    _same_grid(mu, nu)
    start = time.perf_counter()
    rep = quantized_bounds(mu.mass[None, :], nu.mass[None, :], mu.grid.dims, int(kappa),
                           float(p), methods=(method,), return_exceptions=False, **kw)[0][method]
    return rep.__class__(rep.method, rep.value, rep.raw_value, rep.components,
                         time.perf_counter() - start, rep.iterations, rep.coarse_size)


def weighted_cost_upper_bound(mu: GridMeasure, nu: GridMeasure, kappa: int, p: float,
                              precision: str = "fp64"):
    """Coarse LP under C-bar, value^(1/p) (quantized.py:172-196)."""
    return _one(mu, nu, kappa, p, "weighted_cost", precision=precision)


def min_cost_lower_bound(mu: GridMeasure, nu: GridMeasure, kappa: int, p: float,
                         precision: str = "fp64"):
    """Coarse LP under C-min, signed root clipped at 0 (quantized.py:199-223)."""
    return _one(mu, nu, kappa, p, "min_cost", precision=precision)


def primal_upscaling_upper_bound(mu: GridMeasure, nu: GridMeasure, kappa: int, p: float,
                                 xi: float | None = None, kernel: UpscaleKernel | None = None,
                                 max_iter: int = 10_000, precision: str = "fp64"):
    """Upscale the C-tilde plan, IPF-refit, price, add TV terms (quantized.py:288-380)."""
    return _one(mu, nu, kappa, p, "primal_upscaling", xi=xi, kernel=kernel, max_iter=max_iter,
                precision=precision)


def dual_upscaling_lower_bound(mu: GridMeasure, nu: GridMeasure, kappa: int, p: float,
                               method: str = "multilinear", precision: str = "fp64"):
    """Interpolated coarse potential + two fine c-transforms (quantized.py:487-521)."""
    if method not in ("multilinear", "nearest"):
        raise ValueError(f"unknown interpolation method {method!r}")
    return _one(mu, nu, kappa, p, "dual_upscaling", dual_method=method, precision=precision)


def interpolate_potential(coarse_f: np.ndarray, centers: np.ndarray, fine_grid: GridSpec,
                          method: str = "multilinear") -> np.ndarray:
    """Extend a potential from a full centre lattice to the fine grid (device K8)."""
    vals = np.asarray(coarse_f, dtype=np.float64)
    pts = np.asarray(centers, dtype=np.float64)
    d = fine_grid.ndim
    if pts.ndim != 2 or pts.shape[1] != d:
        raise DimensionMismatchError(f"centers must be (n, {d}), got {pts.shape}")
    if vals.shape != (pts.shape[0],):
        raise DimensionMismatchError(
            f"{vals.shape[0] if vals.ndim else 0} values for {pts.shape[0]} centers")
    axes = [np.unique(pts[:, a]) for a in range(d)]
    cdims = tuple(ax.size for ax in axes)
    if int(np.prod(cdims)) != pts.shape[0]:
        raise DimensionMismatchError("centers do not form a full lattice")
    if method not in ("multilinear", "nearest"):
        raise ValueError(f"unknown interpolation method {method!r}")
    device()
    t = torch()
    coarse = to_dev(vals[None, :])
    ax_d = to_dev(np.concatenate(axes))
    out = t.empty((1, fine_grid.cell_count), dtype=t.float64, device=coarse.device)
    N.check(N.lib().gdt_interpolate(N.ptr(coarse), N.ptr(out), 1, d, N.i64s(fine_grid.dims),
                                    N.i64s(cdims), N.ptr(ax_d), 1 if method == "nearest" else 0,
                                    stream()), "gdt_interpolate")
    return to_host(out)[0]


def c_transform(values: np.ndarray, cost: CostSpec, direction: str = "target",
                block_size: int = 1024) -> np.ndarray:
    """Lazy c-transform on the device (quantized.py:450-484); ``block_size`` is
    accepted for API parity (the device kernel tiles on its own)."""
    v = np.asarray(values, dtype=np.float64)
    if direction not in ("target", "source"):
        raise ValueError(f"direction must be 'source' or 'target', got {direction!r}")
    want = cost.n_source if direction == "target" else cost.n_target
    side = "source" if direction == "target" else "target"
    if v.shape != (want,):
        raise DimensionMismatchError(f"potential has {v.shape}, cost has {want} {side} points")
    device()
    t = torch()
    xs, xt, vd = to_dev(cost.source), to_dev(cost.target), to_dev(v)
    n_out = cost.n_target if direction == "target" else cost.n_source
    out = t.empty(n_out, dtype=t.float64, device=vd.device)
    N.check(N.lib().gdt_ctransform_points(N.ptr(xs), N.ptr(xt), cost.n_source, cost.n_target,
                                          cost.source.shape[1], cost.p, N.ptr(vd),
                                          0 if direction == "target" else 1, N.ptr(out),
                                          stream()), "gdt_ctransform_points")
    return to_host(out)
