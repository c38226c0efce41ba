"""Grid measures and their coarsening (reference: pkg/src/gridot/measures.py).

Host side: the frozen data model (``GridSpec``, ``GridMeasure``,
``CoarseningSpec``), the GRID text format (``load_grid_measure`` /
``dump_grid_measure``, measures.py:138-220), index/coordinate helpers and the
closed-form TV weights.  Device side (libgridot_b200.so): SumPool (``coarsen_measure``,
K1, bit-exact with the reference's ``np.add.at`` order), zero padding and
the weighted-TV reduction.

Flat order is axis-1-fastest with 1-based integer coordinates
(measures.py:3-6); block centres are kappa*b + (kappa+1)/2 (measures.py:270-281).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .device import device, stream, to_dev, to_host, torch
from .errors import (DimensionMismatchError, GridFormatError, GridMismatchError,
                     NegativeMassError, ZeroTotalMassError)

__all__ = ["GridSpec", "GridMeasure", "CoarseningSpec", "normalize", "pad_measure",
           "coarsen_measure", "coarsen_grid", "block_index_map", "tv_weights", "weighted_tv",
           "pad_batch", "sumpool_batch", "load_grid_measure", "dump_grid_measure"]


@dataclass(frozen=True)
class GridSpec:
    """Regular grid [1..N_1] x ... x [1..N_d] with unit spacing (measures.py:45-77)."""

    dims: tuple

    def __post_init__(self):
        dims = tuple(int(x) for x in self.dims)
        if not dims:
            raise DimensionMismatchError("a grid needs at least one axis")
        if min(dims) < 1:
            raise DimensionMismatchError(f"grid dims must be positive, got {dims}")
        object.__setattr__(self, "dims", dims)

    @property
    def ndim(self) -> int:
        return len(self.dims)

    @property
    def cell_count(self) -> int:
        return int(np.prod(self.dims))

    def coordinates(self) -> np.ndarray:
        """(cell_count, ndim) float64 coordinates in flat order."""
        axes = np.unravel_index(np.arange(self.cell_count), self.dims, order="F")
        return np.column_stack(axes).astype(np.float64) + 1.0

    def center(self) -> np.ndarray:
        return (np.asarray(self.dims, dtype=np.float64) + 1.0) / 2.0


@dataclass(frozen=True, eq=False)
class GridMeasure:
    """Nonnegative finite masses on the cells of a grid (measures.py:80-109)."""

    grid: GridSpec
    mass: np.ndarray = field(repr=False)

    def __post_init__(self):
        m = np.ascontiguousarray(self.mass, dtype=np.float64)
        if m.ndim != 1 or m.size != self.grid.cell_count:
            raise DimensionMismatchError(
                f"mass vector of length {m.size} does not match {self.grid.cell_count} cells")
        if not np.isfinite(m).all():
            raise ValueError("mass entries must be finite")
        bad = np.flatnonzero(m < 0.0)
        if bad.size:
            raise NegativeMassError(int(bad[0]), float(m[bad[0]]))
        object.__setattr__(self, "mass", m)

    @property
    def total_mass(self) -> float:
        return float(np.sum(self.mass))

    @property
    def support(self) -> np.ndarray:
        return np.flatnonzero(self.mass > 0.0)


# ---------------------------------------------------------------------------
# GRID text format (measures.py:138-220)
# ---------------------------------------------------------------------------


def _grid_text(source) -> str:
    if isinstance(source, bytes):
        return source.decode("ascii", errors="replace")
    if isinstance(source, str):
        return source
    if hasattr(source, "read"):
        raw = source.read()
        return raw.decode("ascii", errors="replace") if isinstance(raw, bytes) else raw
    raise TypeError(f"cannot read GRID data from {type(source).__name__}")


def load_grid_measure(source) -> GridMeasure:
    """Parse GRID text: '#' comment and blank lines, a header ``d N1 .. Nd``,
    then exactly N1*..*Nd whitespace-separated masses in flat order (axis 1
    fastest).  Accepts str, bytes or a file object (measures.py:138-204).

    Failures raise GridFormatError with the 1-based line of the header (or
    of the first body line for count errors) and the 0-based index of a bad
    mass token, or NegativeMassError with the flat index of the first
    negative entry -- the reference's checks, in its order.
    """
    lines = _grid_text(source).split("\n")
    hno = next((no for no, ln in enumerate(lines, start=1)
                if ln.strip() and not ln.strip().startswith("#")), None)
    if hno is None:
        raise GridFormatError("no header line found")
    header = lines[hno - 1].strip()
    head = header.split()
    try:
        d = int(head[0])
    except ValueError:
        raise GridFormatError(f"dimension count {head[0]!r} is not an integer", line=hno)
    if d < 1:
        raise GridFormatError(f"dimension count must be >= 1, got {d}", line=hno)
    if len(head) != d + 1:
        raise GridFormatError(f"header needs {d + 1} integers for d={d}, got {len(head)}",
                              line=hno)
    try:
        dims = tuple(int(tok) for tok in head[1:])
    except ValueError:
        raise GridFormatError(f"bad axis length in header {header!r}", line=hno)
    if min(dims) < 1:
        raise GridFormatError(f"axis lengths must be positive, got {dims}", line=hno)
    grid = GridSpec(dims)
    tokens = "\n".join(lines[hno:]).split()
    if len(tokens) != grid.cell_count:
        raise GridFormatError(f"expected {grid.cell_count} mass entries, got {len(tokens)}",
                              line=hno + 1)
    try:  # Python's float() grammar, as the reference parses each token
        mass = np.fromiter(map(float, tokens), dtype=np.float64, count=len(tokens))
    except ValueError:
        for i, tok in enumerate(tokens):
            try:
                float(tok)
            except ValueError:
                raise GridFormatError(f"bad mass entry {tok!r}", token=i) from None
        raise
    bad = np.flatnonzero(~np.isfinite(mass))
    if bad.size:
        raise GridFormatError(f"non-finite mass entry {tokens[bad[0]]!r}", token=int(bad[0]))
    neg = np.flatnonzero(mass < 0.0)
    if neg.size:
        raise NegativeMassError(int(neg[0]), float(mass[neg[0]]))
    return GridMeasure(grid, mass)


def dump_grid_measure(measure: GridMeasure) -> str:
    """GRID text with round-tripping float reprs, one axis-1 run per line
    (measures.py:207-216)."""
    dims = measure.grid.dims
    n1 = dims[0]
    m = measure.mass
    rows = (" ".join(map(repr, m[i:i + n1].tolist())) for i in range(0, m.size, n1))
    return f"{len(dims)} " + " ".join(map(str, dims)) + "\n" + "\n".join(rows) + "\n"


@dataclass(frozen=True)
class CoarseningSpec:
    """Block edge length kappa (measures.py:112-130)."""

    kappa: int

    def __post_init__(self):
        k = int(self.kappa)
        if k < 1:
            raise ValueError(f"kappa must be >= 1, got {self.kappa}")
        object.__setattr__(self, "kappa", k)

    def padded_dims(self, grid: GridSpec) -> tuple:
        k = self.kappa
        return tuple(-(-n // k) * k for n in grid.dims)

    def coarse_dims(self, grid: GridSpec) -> tuple:
        return tuple(n // self.kappa for n in self.padded_dims(grid))


def normalize(measure: GridMeasure) -> GridMeasure:
    total = measure.total_mass
    if total <= 0.0:
        raise ZeroTotalMassError("cannot normalize a measure with zero total mass")
    return GridMeasure(measure.grid, measure.mass / total)


def block_index_map(grid: GridSpec, coarsening: CoarseningSpec) -> np.ndarray:
    """Coarse flat id of every fine cell (measures.py:248-254)."""
    k = coarsening.kappa
    axes = np.unravel_index(np.arange(grid.cell_count), grid.dims, order="F")
    return np.ravel_multi_index(tuple(a // k for a in axes), coarsening.coarse_dims(grid),
                                order="F")


def coarsen_grid(grid: GridSpec, coarsening: CoarseningSpec) -> np.ndarray:
    """Block centres (n_coarse, ndim) in coarse flat order."""
    cd = coarsening.coarse_dims(grid)
    k = coarsening.kappa
    axes = np.unravel_index(np.arange(int(np.prod(cd))), cd, order="F")
    return np.column_stack(axes).astype(np.float64) * k + (k + 1) / 2.0


def tv_weights(grid: GridSpec, p: float, metric: str = "l2") -> np.ndarray:
    """rho(centre, x_i)^p per cell (measures.py:289-295); host closed form."""
    if metric != "l2":
        raise ValueError(f"unsupported metric {metric!r}")
    diff = grid.coordinates() - grid.center()[None, :]
    return np.sum(diff * diff, axis=1) ** (p / 2.0)


# ---------------------------------------------------------------------------
# device entry points
# ---------------------------------------------------------------------------


def pad_batch(x, dims, kappa):
    """[B, prod(dims)] device tensor -> zero-padded [B, prod(padded)] (K: gdt_pad_f64)."""
    pd = tuple(-(-n // kappa) * kappa for n in dims)
    if pd == tuple(dims):
        return x, pd
    out = torch().empty((x.shape[0], int(np.prod(pd))), dtype=torch().float64, device=x.device)
    N.check(N.lib().gdt_pad_f64(N.ptr(x), N.ptr(out), x.shape[0], len(dims), N.i64s(dims),
                                kappa, stream()), "gdt_pad_f64")
    return out, pd


def sumpool_batch(x, dims, kappa, stats=None):
    """[B, prod(dims)] -> [B, n_coarse] block sums on the device (bit-exact order).

    ``stats`` (a [B, n_coarse, 3] float64 device tensor) also receives each
    block's smallest / largest positive mass and positive-cell count from the
    same pass (gdt_sumpool_stats_f64)."""
    xp, pd = pad_batch(x, dims, kappa)
    ops = N.torch_ops()
    if ops is not None:  # the PyTorch extension's operator (same C entry point)
        return ops.sumpool(xp.contiguous(), [int(d) for d in pd], int(kappa), stats)
    nc = int(np.prod(pd)) // kappa ** len(dims)
    out = torch().empty((x.shape[0], nc), dtype=torch().float64, device=x.device)
    N.check(N.lib().gdt_sumpool_stats_f64(N.ptr(xp), N.ptr(out), N.ptr(stats), x.shape[0],
                                          len(dims), N.i64s(pd), kappa, stream()),
            "gdt_sumpool_stats_f64")
    return out


def pad_measure(measure: GridMeasure, coarsening: CoarseningSpec) -> GridMeasure:
    """Zero-pad to a kappa multiple (measures.py:236-245), on the device."""
    pd = coarsening.padded_dims(measure.grid)
    if pd == measure.grid.dims:
        return measure
    x = to_dev(measure.mass[None, :])
    out, _ = pad_batch(x, measure.grid.dims, coarsening.kappa)
    return GridMeasure(GridSpec(pd), to_host(out)[0])


def coarsen_measure(measure: GridMeasure, coarsening: CoarseningSpec) -> GridMeasure:
    """SumPool on the device (measures.py:257-267)."""
    out = sumpool_batch(to_dev(measure.mass[None, :]), measure.grid.dims, coarsening.kappa)
    return GridMeasure(GridSpec(coarsening.coarse_dims(measure.grid)), to_host(out)[0])


def weighted_tv(a: GridMeasure, b: GridMeasure, weights: np.ndarray, p: float) -> float:
    """2^(1-1/p) (sum_i w_i |a_i - b_i|)^(1/p) (measures.py:298-315); the
    weighted sum runs on the device."""
    if a.grid != b.grid:
        raise GridMismatchError(f"grids differ: {a.grid.dims} vs {b.grid.dims}")
    w = np.asarray(weights, dtype=np.float64)
    if w.shape != a.mass.shape:
        raise DimensionMismatchError(
            f"weight vector of length {w.size} does not match {a.mass.size} cells")
    device()
    xa, xb, wd = to_dev(a.mass[None, :]), to_dev(b.mass[None, :]), to_dev(w)
    out = torch().empty(1, dtype=torch().float64, device=xa.device)
    N.check(N.lib().gdt_weighted_tv_inner(N.ptr(xa), N.ptr(xb), 1, a.grid.ndim,
                                          N.i64s(a.grid.dims), float(p), N.ptr(wd), N.ptr(out),
                                          stream()), "gdt_weighted_tv_inner")
    inner = float(to_host(out)[0])
    return 2.0 ** (1.0 - 1.0 / p) * inner ** (1.0 / p)
