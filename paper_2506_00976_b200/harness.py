"""Batched bench matrix and CSV report on the device path (reference `cli.py`).

Mirrors the reference's reporting contract so its CSV consumers carry over:
``CSV_COLUMNS`` / ``ReportRow`` (cli.py:46-49, 170-193), ``gen_synthetic``
(cli.py:60-103), ``BenchConfig`` (cli.py:116-167), ``bench_run`` /
``write_csv`` (cli.py:282-310), the ``bench`` sub-command (cli.py:335-356) and
the ``dist`` sub-command (cli.py:358-445: two GRID files, one method, one CSV
record on stdout).

Differences, all deliberate:
* the quantization bounds of all pairs of one class run as ONE batched device
  call per (p, kappa) (``engine.quantized_bounds``); a row's ``wall_time`` is
  that call's wall time divided by the number of pairs;
* the exact baseline is the host network simplex (same pivot rules as
  ``_simplex.py``) on the fine grid with an offset-table cost, all pairs of a
  class in one multi-threaded batch;
* the entropic methods (``reg_lower``, ``reg_upper``, sinkhorn.py:150-299) run
  per pair on the device (``sinkhorn.reg_lower_bound`` / ``reg_upper_bound``)
  with epsilon = multiplier * n^p (cli.py:224-232), one row per ``--eps``
  multiplier.
"""

from __future__ import annotations

import argparse
import csv
import io
import logging
import sys
import time
from dataclasses import dataclass

import numpy as np

from .costs import CostSpec, centre_cost_table
from .engine import QUANT_METHODS, quantized_bounds
from .errors import GridotError
from .exact import build_transport_problem, solve_transport_many
from .measures import GridMeasure, GridSpec, load_grid_measure, normalize
from .sinkhorn import RegularizationParams, reg_lower_bound, reg_upper_bound

logger = logging.getLogger(__name__)

GENERATOR_CLASSES = ("gaussians", "shapes", "noise")
REG_METHODS = ("reg_lower", "reg_upper")
LOWER_METHODS = frozenset({"min_cost", "dual_upscaling", "reg_lower"})
ALL_METHODS = ("exact",) + QUANT_METHODS + REG_METHODS
SUPPORTED_METHODS = ALL_METHODS
MAX_EXACT_CELLS = 2 ** 16  # the reference's bench limit (sinkhorn.MAX_KERNEL_CELLS)

CSV_COLUMNS = (
    "pair", "method", "p", "param", "bound", "exact",
    "rel_error", "wall_time", "rel_time", "error",
)


class CliValidationError(GridotError):
    """Bad command-line arguments or configuration."""


# ---------------------------------------------------------------------------
# synthetic measures (cli.py:60-103): the same generator classes and the same
# sequence of draws from numpy's default_rng, so a seed gives the same measure
# ---------------------------------------------------------------------------


def _coordinates(n: int, d: int) -> np.ndarray:
    return GridSpec((n,) * d).coordinates()


def gen_synthetic(kind: str, n: int, d: int, seed) -> GridMeasure:
    if n < 4:
        raise CliValidationError(f"generator needs n >= 4, got {n}")
    if d < 1:
        raise CliValidationError(f"generator needs d >= 1, got {d}")
    if kind not in GENERATOR_CLASSES:
        raise CliValidationError(
            f"unknown generator {kind!r}; choose from {', '.join(GENERATOR_CLASSES)}")
    rng = np.random.default_rng(seed)
    grid = GridSpec((n,) * d)
    x = _coordinates(n, d)
    cells = x.shape[0]
    dens = np.zeros(cells)
    if kind == "noise":
        dens = rng.uniform(0.05, 1.0, size=cells)
    elif kind == "gaussians":
        for _ in range(int(rng.integers(1, 4))):
            c = rng.uniform(1.0, n, size=d)
            s = rng.uniform(n / 16.0, n / 4.0)
            w = rng.uniform(0.2, 1.0)
            r2 = np.sum((x - c[None, :]) ** 2, axis=1)
            dens += w * np.exp(-r2 / (2.0 * s ** 2))
    else:  # shapes: boxes or balls of constant fill
        for _ in range(int(rng.integers(1, 4))):
            fill = rng.uniform(0.5, 1.5)
            if rng.random() < 0.5:
                u = rng.uniform(1.0, n, size=d)
                v = rng.uniform(1.0, n, size=d)
                mask = np.all((x >= np.minimum(u, v)) & (x <= np.maximum(u, v)), axis=1)
            else:
                c = rng.uniform(1.0, n, size=d)
                rad = rng.uniform(n / 8.0, n / 3.0)
                mask = np.sum((x - c[None, :]) ** 2, axis=1) <= rad * rad
            dens[mask] += fill
        if dens.sum() <= 0.0:
            dens[cells // 2] = 1.0
    return normalize(GridMeasure(grid, dens))


# ---------------------------------------------------------------------------
# configuration and rows
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class BenchConfig:
    classes: tuple = ("gaussians",)
    n: int = 32
    d: int = 2
    p_values: tuple = (1.0, 2.0)
    kappas: tuple = (2, 4)
    xi: float | None = None
    seed: int = 0
    n_pairs: int = 3
    methods: tuple = SUPPORTED_METHODS
    out: str | None = None
    max_iter: int = 10_000
    precision: str = "fp64"
    eps_multipliers: tuple = (0.001, 0.004)

    def validate(self) -> None:
        for cls in self.classes:
            if cls not in GENERATOR_CLASSES:
                raise CliValidationError(f"unknown generator class {cls!r}")
        if self.n < 4:
            raise CliValidationError(f"n must be >= 4, got {self.n}")
        if self.d < 1:
            raise CliValidationError(f"d must be >= 1, got {self.d}")
        if self.n ** self.d > MAX_EXACT_CELLS:
            raise CliValidationError(
                f"n^d = {self.n ** self.d} exceeds {MAX_EXACT_CELLS}; "
                "the bench always solves the exact baseline per pair")
        for p in self.p_values:
            if p < 1.0:
                raise CliValidationError(f"p must be >= 1, got {p}")
        for k in self.kappas:
            if k < 1:
                raise CliValidationError(f"kappa must be >= 1, got {k}")
        if self.xi is not None and self.xi <= 0.0:
            raise CliValidationError(f"xi must be > 0, got {self.xi}")
        if self.n_pairs < 1:
            raise CliValidationError(f"pairs must be >= 1, got {self.n_pairs}")
        if not self.methods:
            raise CliValidationError("no methods selected")
        for m in self.eps_multipliers:
            if m <= 0.0:
                raise CliValidationError(f"eps multiplier must be > 0, got {m}")
        for m in self.methods:
            if m not in ALL_METHODS:
                raise CliValidationError(
                    f"unknown method {m!r}; choose from {', '.join(SUPPORTED_METHODS)}")
        if self.max_iter < 1:
            raise CliValidationError(f"max-iter must be >= 1, got {self.max_iter}")
        if self.precision not in ("fp64", "fp32"):
            raise CliValidationError(f"precision must be fp64 or fp32, got {self.precision!r}")


@dataclass
class ReportRow:
    """One CSV row; numeric fields are None when unavailable."""

    pair: str
    method: str
    p: float
    param: str = ""
    bound: float | None = None
    exact: float | None = None
    rel_error: float | None = None
    wall_time: float | None = None
    rel_time: float | None = None
    error: str = ""

    def as_record(self) -> list:
        def num(v):
            return "" if v is None else format(v, ".17g")

        return [self.pair, self.method, num(self.p), self.param, num(self.bound),
                num(self.exact), num(self.rel_error), num(self.wall_time), num(self.rel_time),
                self.error]


def _relative_error(method: str, bound: float, exact):
    if exact is None:
        return None
    if method == "exact":
        return 0.0
    scale = exact if exact != 0.0 else 1.0
    return (exact - bound) / scale if method in LOWER_METHODS else (bound - exact) / scale


# ---------------------------------------------------------------------------
# the matrix
# ---------------------------------------------------------------------------


def exact_distances(mus, nus, n: int, d: int, p: float, threads: int = 0):
    """W_p of every pair on the fine grid (exact.py:139-189), one LP batch.

    Returns a list of (value or None, wall seconds per pair, error text)."""
    table = centre_cost_table((n,) * d, 1, float(p))  # kappa = 1: the fine costs
    probs, errs = [], []
    for mu, nu in zip(mus, nus):
        try:
            probs.append(build_transport_problem(mu, nu, table))
            errs.append(None)
        except GridotError as exc:
            probs.append(None)
            errs.append(f"{type(exc).__name__}: {exc}")
    live = [q for q in probs if q is not None]
    t0 = time.perf_counter()
    solved = iter(solve_transport_many(live, threads=threads, slack=False))
    per = (time.perf_counter() - t0) / max(1, len(live))
    out = []
    for q, e in zip(probs, errs):
        if q is None:
            out.append((None, None, e))
            continue
        r = next(solved)
        if isinstance(r, Exception):
            out.append((None, None, f"{type(r).__name__}: {r}"))
        else:
            out.append((r[2] ** (1.0 / p), per, ""))
    return out


def _class_rows(cls: str, class_index: int, cfg: BenchConfig) -> list:
    mus, nus, ids = [], [], []
    for pair_index in range(cfg.n_pairs):
        mus.append(gen_synthetic(cls, cfg.n, cfg.d, seed=[cfg.seed, class_index, pair_index, 0]))
        nus.append(gen_synthetic(cls, cfg.n, cfg.d, seed=[cfg.seed, class_index, pair_index, 1]))
        ids.append(f"{cls}-{pair_index:03d}")
    dims = (cfg.n,) * cfg.d
    mu_mat = np.stack([m.mass for m in mus])
    nu_mat = np.stack([m.mass for m in nus])
    quant = [m for m in cfg.methods if m in QUANT_METHODS]
    rows = []
    for p in cfg.p_values:
        exact = exact_distances([m.mass for m in mus], [m.mass for m in nus], cfg.n, cfg.d, p)
        for i, pid in enumerate(ids):
            value, wall, err = exact[i]
            if err:
                logger.warning("exact baseline failed on %s (p=%g): %s", pid, p, err)
            if "exact" in cfg.methods:
                rows.append(ReportRow(pid, "exact", p, bound=value, exact=value,
                                      rel_error=0.0 if value is not None else None,
                                      wall_time=wall,
                                      rel_time=1.0 if wall is not None else None, error=err))
        for k in cfg.kappas:
            if not quant:
                continue
            t0 = time.perf_counter()
            try:
                reps = quantized_bounds(mu_mat, nu_mat, dims, int(k), float(p),
                                        precision=cfg.precision, xi=cfg.xi,
                                        max_iter=cfg.max_iter, methods=tuple(quant),
                                        return_exceptions=True)
                batch_err = None
            except GridotError as exc:
                reps, batch_err = None, f"{type(exc).__name__}: {exc}"
            wall = (time.perf_counter() - t0) / len(ids)
            for i, pid in enumerate(ids):
                ex_value, ex_wall, _ = exact[i]
                for m in quant:
                    row = ReportRow(pid, m, p, param=str(k), exact=ex_value)
                    res = reps[i][m] if reps is not None else None
                    if batch_err is not None or isinstance(res, Exception):
                        row.error = batch_err or f"{type(res).__name__}: {res}"
                        logger.warning("%s failed on %s (p=%g, param=%s): %s", m, pid, p, k,
                                       row.error)
                    else:
                        row.bound = res.value
                        row.wall_time = wall
                        row.rel_error = _relative_error(m, res.value, ex_value)
                        if ex_wall:
                            row.rel_time = wall / ex_wall
                    rows.append(row)
        reg = [m for m in cfg.methods if m in REG_METHODS]
        coords = GridSpec(dims).coordinates()
        for i, pid in enumerate(ids):
            ex_value, ex_wall, _ = exact[i]
            for m in reg:
                fn = reg_lower_bound if m == "reg_lower" else reg_upper_bound
                for mult in cfg.eps_multipliers:
                    row = ReportRow(pid, m, p, param=format(mult, "g"), exact=ex_value)
                    try:
                        params = RegularizationParams(epsilon=mult * max(dims) ** p, xi=cfg.xi,
                                                      max_iter=cfg.max_iter)
                        rep = fn(mus[i], nus[i], CostSpec(coords, coords, p), params)
                        row.bound, row.wall_time = rep.value, rep.wall_time
                        row.rel_error = _relative_error(m, rep.value, ex_value)
                        if ex_wall:
                            row.rel_time = rep.wall_time / ex_wall
                    except GridotError as exc:
                        row.error = f"{type(exc).__name__}: {exc}"
                        logger.warning("%s failed on %s (p=%g, param=%s): %s", m, pid, p,
                                       row.param, exc)
                    rows.append(row)
    return rows


def bench_run(cfg: BenchConfig) -> list:
    """The bench matrix; rows sorted by (pair, method, param) like cli.bench_run."""
    cfg.validate()
    rows = []
    for ci, cls in enumerate(cfg.classes):
        rows.extend(_class_rows(cls, ci, cfg))
    rows.sort(key=lambda r: (r.pair, r.method, r.param))
    return rows


def write_csv(rows, stream) -> None:
    w = csv.writer(stream, lineterminator="\n")
    w.writerow(CSV_COLUMNS)
    for r in rows:
        w.writerow(r.as_record())


def rows_to_csv(rows) -> str:
    buf = io.StringIO()
    write_csv(rows, buf)
    return buf.getvalue()


def _exact_one(mu: GridMeasure, nu: GridMeasure, p: float):
    """W_p on the fine grid by the host simplex (exact.py:139-189); (value, s)."""
    table = centre_cost_table(mu.grid.dims, 1, float(p))  # kappa = 1: the fine costs
    t0 = time.perf_counter()
    (res,) = solve_transport_many([build_transport_problem(mu.mass, nu.mass, table)],
                                  threads=1, slack=False)
    if isinstance(res, Exception):
        raise res
    return res[2] ** (1.0 / p), time.perf_counter() - t0


def dist_run(mu_path: str, nu_path: str, method: str, p: float = 2.0, kappa: int = 2,
             eps: float = 0.001, xi=None, max_iter: int = 10_000,
             precision: str = "fp64") -> ReportRow:
    """One bound between two GRID files (cli.py:398-445); GridotError raised by
    the method is recorded in the row's ``error``."""
    if method not in ALL_METHODS:
        raise CliValidationError(
            f"unknown method {method!r}; choose from {', '.join(ALL_METHODS)}")
    if p < 1.0:
        raise CliValidationError(f"p must be >= 1, got {p}")
    with open(mu_path) as fh:
        mu = normalize(load_grid_measure(fh))
    with open(nu_path) as fh:
        nu = normalize(load_grid_measure(fh))
    if mu.grid != nu.grid:
        raise CliValidationError(
            f"measures live on different grids: {mu.grid.dims} vs {nu.grid.dims}")
    param = "" if method == "exact" else (format(eps, "g") if method in REG_METHODS
                                          else str(kappa))
    row = ReportRow(pair="dist", method=method, p=p, param=param)
    try:
        if method == "exact":
            value, wall = _exact_one(mu, nu, p)
            row.exact, row.rel_error, row.rel_time = value, 0.0, 1.0
        elif method in REG_METHODS:
            fn = reg_lower_bound if method == "reg_lower" else reg_upper_bound
            coords = mu.grid.coordinates()
            rep = fn(mu, nu, CostSpec(coords, coords, p),
                     RegularizationParams(epsilon=eps * max(mu.grid.dims) ** p, xi=xi,
                                          max_iter=max_iter))
            value, wall = rep.value, rep.wall_time
        else:
            reps = quantized_bounds(mu.mass[None], nu.mass[None], mu.grid.dims, int(kappa),
                                    float(p), precision=precision, xi=xi, max_iter=max_iter,
                                    methods=(method,), return_exceptions=False)
            value, wall = reps[0][method].value, reps[0][method].wall_time
        row.bound, row.wall_time = value, wall
    except GridotError as exc:
        row.error = f"{type(exc).__name__}: {exc}"
    return row


# ---------------------------------------------------------------------------
# command line: python -m paper_2506_00976_b200.harness bench ...
# ---------------------------------------------------------------------------


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        raise CliValidationError(message)


def _split(text: str, cast):
    try:
        return tuple(cast(tok) for tok in text.split(",") if tok)
    except ValueError as exc:
        raise CliValidationError(f"cannot parse list {text!r}: {exc}")


def _parser() -> _Parser:
    ap = _Parser(prog="gridot-b200", description=__doc__,
                 formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("-v", "--verbose", action="count", default=0)
    sub = ap.add_subparsers(dest="command", required=True)
    b = sub.add_parser("bench", help="run the synthetic benchmark matrix on the device")
    b.add_argument("--class", dest="classes", default="gaussians")
    b.add_argument("--n", type=int, default=32)
    b.add_argument("--d", type=int, default=2)
    b.add_argument("--p", default="1,2")
    b.add_argument("--kappa", default="2,4")
    b.add_argument("--xi", type=float, default=None)
    b.add_argument("--pairs", type=int, default=3)
    b.add_argument("--seed", type=int, default=0)
    b.add_argument("--methods", default="all")
    b.add_argument("--max-iter", type=int, default=10_000)
    b.add_argument("--precision", default="fp64")
    b.add_argument("--eps", default="0.001,0.004")
    b.add_argument("--out", default=None)
    d = sub.add_parser("dist", help="bound the distance between two GRID files")
    d.add_argument("--mu", required=True)
    d.add_argument("--nu", required=True)
    d.add_argument("--method", required=True)
    d.add_argument("--p", type=float, default=2.0)
    d.add_argument("--kappa", type=int, default=2)
    d.add_argument("--eps", type=float, default=0.001)
    d.add_argument("--xi", type=float, default=None)
    d.add_argument("--max-iter", type=int, default=10_000)
    d.add_argument("--precision", default="fp64")
    return ap


def main(argv=None) -> int:
    try:
        args = _parser().parse_args(argv)
        level = (logging.WARNING, logging.INFO, logging.DEBUG)[min(args.verbose, 2)]
        logging.basicConfig(level=level, format="%(levelname)s %(name)s: %(message)s")
        if args.command == "dist":
            row = dist_run(args.mu, args.nu, args.method, args.p, args.kappa, args.eps, args.xi,
                           args.max_iter, args.precision)
            print(",".join(row.as_record()))
            if row.error:
                print(f"gridot-b200: {row.error}", file=sys.stderr)
                return 2
            return 0
        methods = (SUPPORTED_METHODS if args.methods.strip() == "all"
                   else _split(args.methods, str))
        cfg = BenchConfig(classes=_split(args.classes, str), n=args.n, d=args.d,
                          p_values=_split(args.p, float), kappas=_split(args.kappa, int),
                          xi=args.xi, seed=args.seed, n_pairs=args.pairs, methods=methods,
                          out=args.out, max_iter=args.max_iter, precision=args.precision,
                          eps_multipliers=_split(args.eps, float))
        rows = bench_run(cfg)
        if cfg.out is None:
            write_csv(rows, sys.stdout)
        else:
            with open(cfg.out, "w", newline="") as fh:
                write_csv(rows, fh)
            logger.info("wrote %d rows to %s", len(rows), cfg.out)
        return 0
    except CliValidationError as exc:
        print(f"gridot-b200: {exc}", file=sys.stderr)
        return 1
    except (OSError, GridotError) as exc:
        print(f"gridot-b200: {type(exc).__name__}: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
