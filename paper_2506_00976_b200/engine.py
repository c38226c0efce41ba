"""Batched quantization-bound engine: B pairs x one (kappa, p) per call.

Unit of work = one pair (mu, nu) at one (kappa, p), producing the four bounds
of ``QUANT_METHODS`` (reference cli.py:41).  Per batch the device does

    H2D(mu, nu) -> pad -> SumPool (K1) -> C-bar (K2) -> D2H(mu~, nu~, C-bar)
    host: coarse LPs (C-tilde, C-bar, C-min) on a native thread pool
    H2D(arcs, duals) -> primal upscaling IPF + pricing + TV (K4-K6)
                     -> coarse c-transform (K7) -> interpolation (K8)
                     -> two c-transforms + dual dots (K9, K10)
    D2H(per-pair scalars)

and the host turns the scalars into ``BoundReport`` objects with exactly the
reference's final arithmetic (``** (1/p)``, ``signed_root``, clipping).

``prepare_coarse`` + ``gpu_stages`` split the pipeline at the LP boundary so
the benchmark can time the device stages with coarse plans precomputed
(SURVEY.md 8(d) "GPU-stage throughput").
"""

from __future__ import annotations

import threading
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .costs import (centre_cost_cached, centre_cost_table, cost_table, max_sq_of,
                    min_cost_table, weighted_cost_batch)
from .device import device, pinned_empty, stream, to_dev, to_host, to_host_pinned, torch
from .errors import DimensionMismatchError, GridotError, NumericOverflowError, \
    ZeroDenominatorError
from .exact import LPBatch, TransportProblem, build_transport_problem, solve_transport_many
from .measures import (CoarseningSpec, GridSpec, block_index_map, coarsen_grid, pad_batch,
                       sumpool_batch, tv_weights)
from .reports import BoundReport, signed_root

__all__ = ["QUANT_METHODS", "CoarsePlans", "DevicePlans", "quantized_bounds", "prepare_coarse",
           "gpu_stages", "PRECISIONS", "make_batch"]

QUANT_METHODS = ("weighted_cost", "min_cost", "primal_upscaling", "dual_upscaling")
PRECISIONS = ("fp64", "fp32")
_MODE = {"fp64": 0, "fp32": 1}


def _uniform_paired(kappa: int, d: int) -> np.ndarray:
    m = kappa ** d
    w = np.full((kappa,) * (2 * d), 1.0 / (kappa ** (2 * d)))
    w = w / float(w.sum())
    return w.reshape((m, m), order="F")


@dataclass
class CoarsePlans:
    """Host-side LP results for a batch (one entry per pair)."""

    n: int
    ctil_arcs: list = field(default_factory=list)     # (rows, cols, mass) full coarse ids
    ctil_duals: list = field(default_factory=list)    # (g, dst_index)
    ctil_error: list = field(default_factory=list)
    cbar_value: list = field(default_factory=list)    # float or exception
    cmin_value: list = field(default_factory=list)    # float or exception
    lp_seconds: float = 0.0
    cbar_seconds: float = 0.0    # C-bar kernel + D2H
    table_seconds: float = 0.0   # offset tables
    build_seconds: float = 0.0   # problem construction
    solve_seconds: float = 0.0   # the native LP batch


class _Batch:
    """Device state of one batch at one (kappa, p)."""

    def __init__(self, mu, nu, dims, kappa, p, precision):
        t = torch()
        self.t = t
        self.dims = tuple(int(x) for x in dims)
        self.d = len(self.dims)
        self.kappa = int(kappa)
        self.p = float(p)
        self.precision = precision
        self.mode = _MODE[precision]
        self.mu = mu
        self.nu = nu
        self.B = mu.shape[0]
        self.dev = mu.device
        self.pdims = tuple(-(-n // self.kappa) * self.kappa for n in self.dims)
        self.cdims = tuple(n // self.kappa for n in self.pdims)
        self.n = int(np.prod(self.cdims))
        self.ctil = centre_cost_cached(self.pdims, self.kappa, self.p)
        self.ctil_dev = to_dev(self.ctil)
        self.table_dev = None
        self.max_sq = 0
        self.cbar_dev = None  # C-bar of the batch once _cbar ran
        if self.p != 2.0:
            self.max_sq = max(max_sq_of(self.pdims), max_sq_of(self.dims))
            self.table_dev = to_dev(cost_table(self.max_sq, self.p))
        self.pool()

    def pool(self):
        """Zero padding + SumPool (K1) of both sides; re-run per step by the bench."""
        self.mu_pad, _ = pad_batch(self.mu, self.dims, self.kappa)
        self.nu_pad, _ = pad_batch(self.nu, self.dims, self.kappa)
        # block statistics of both sides from the same pass (mu then nu): the
        # fp32-mode primal stage works on them instead of the fine masses
        t = self.t
        self.stats = t.empty((2, self.B, self.n, 3), dtype=t.float64, device=self.dev)
        self.mu_c = sumpool_batch(self.mu_pad, self.pdims, self.kappa, self.stats[0])
        self.nu_c = sumpool_batch(self.nu_pad, self.pdims, self.kappa, self.stats[1])


# ---------------------------------------------------------------------------
# stage 1: SumPool, C-bar, host LPs
# ---------------------------------------------------------------------------


def cbar_parent(bt: "_Batch", done, computed: bool = True):
    """A batch among `done` (their C-bar already computed, same masses) whose
    C-bar can be pooled into bt's: fp32 mode, p != 2 (the O(N^2) fp32 kernel),
    the same padded grid and a pooling factor dividing bt's -- the largest such
    factor.  None otherwise."""
    if bt.mode != 1 or bt.p == 2.0:
        return None
    best = None
    for o in done:
        if (o is not bt and (o.cbar_dev is not None or not computed) and o.mode == 1
                and o.p == bt.p
                and o.pdims == bt.pdims and o.B == bt.B and o.kappa < bt.kappa
                and bt.kappa % o.kappa == 0 and (best is None or o.kappa > best.kappa)):
            best = o
    return best


def _cbar(bt: _Batch, parent: "_Batch | None" = None):
    if parent is not None:
        # nested blocks: the numerator of C-bar is additive over the parent's
        # blocks (costs.py:128-171), no second pass over the fine cells
        t = bt.t
        out = t.empty((bt.B, bt.n, bt.n), dtype=t.float64, device=bt.dev)
        N.check(N.lib().gdt_weighted_cost_pool(
            N.ptr(parent.cbar_dev), N.ptr(parent.mu_c), N.ptr(parent.nu_c), N.ptr(bt.mu_c),
            N.ptr(bt.nu_c), N.ptr(bt.ctil_dev), N.ptr(out), None, bt.B, bt.d,
            N.i64s(parent.cdims), bt.kappa // parent.kappa, stream()), "gdt_weighted_cost_pool")
        bt.cbar_dev = out
        return out, None
    # p == 2: C-bar from fp64 block moments in both precisions (the quadratic
    # cost factorises; <= ~1e-14 relative per entry against the reference's
    # summation, far inside fp64 mode's 1e-9 bound contract); p != 2: the
    # reference-order fp64 kernel (fp64 mode) or the fp32 FFMA2 kernel
    mode = 1 if bt.p == 2.0 else bt.mode
    out = weighted_cost_batch(bt.mu_pad, bt.nu_pad, bt.mu_c, bt.nu_c, bt.pdims, bt.kappa, bt.p,
                              mode, bt.ctil_dev, bt.table_dev, want_unused=False)
    bt.cbar_dev = out[0]  # kept: the fp32-mode primal stage prices the fitted plan with it
    return out


@dataclass
class _LPJob:
    """The coarse LPs of one batch at one (kappa, p), before solving."""

    plans: CoarsePlans
    problems: list
    slots: list
    warm: list
    need: tuple
    cbar_host: object = None  # keeps the pinned C-bar alive until the solve


def coarse_problems(bt: _Batch, methods) -> _LPJob:
    """SumPool + C-bar on the device and every coarse LP the methods need."""
    need_ctil = "primal_upscaling" in methods or "dual_upscaling" in methods
    need_cbar = "weighted_cost" in methods
    need_cmin = "min_cost" in methods
    cbar_host = None
    tc = time.perf_counter()
    if need_cbar:
        vals, _ = _cbar(bt)
        cbar_host = to_host_pinned(vals)
    mu_c = to_host(bt.mu_c)
    nu_c = to_host(bt.nu_c)
    plans = CoarsePlans(n=bt.n)
    t0 = time.perf_counter()
    plans.cbar_seconds = t0 - tc
    problems, slots, warm = [], [], []
    # C-tilde and C-min are translation-invariant: the host LP reads offset
    # tables instead of n x n matrices (dense copies only for partial supports)
    cmin = min_cost_table(bt.pdims, bt.kappa, bt.p) if need_cmin else None
    ctil = centre_cost_table(bt.pdims, bt.kappa, bt.p) if need_ctil else None
    plans.table_seconds = time.perf_counter() - t0
    for b in range(bt.B):
        prev = -1
        for kind, cost in (("ctil", ctil),
                           ("cbar", cbar_host[b] if need_cbar else None),
                           ("cmin", cmin)):
            if cost is None:
                continue
            try:
                problems.append(build_transport_problem(mu_c[b], nu_c[b], cost))
                slots.append((b, kind))
                # C-tilde follows the reference's pivot path (its basis defines the
                # upscaled support and the duals); C-bar / C-min only need the
                # optimal value, so each starts from the previous optimal basis of
                # the chain C-tilde -> C-bar -> C-min (same marginals)
                warm.append(prev)
                prev = len(problems) - 1
            except GridotError as exc:
                slots.append((b, kind, exc))
    plans.build_seconds = time.perf_counter() - t0 - plans.table_seconds
    return _LPJob(plans, problems, slots, warm, (need_ctil, need_cbar, need_cmin), cbar_host)


def assemble_plans(bt: _Batch, job: _LPJob, solved) -> CoarsePlans:
    """Per-pair plans / values from the solved LPs of one job."""
    need_ctil, need_cbar, need_cmin = job.need
    plans = job.plans
    res = {}
    it = iter(zip(job.problems, solved))
    for s in job.slots:
        if len(s) == 3:
            res[(s[0], s[1])] = (None, s[2])
        else:
            prob, out = next(it)
            res[(s[0], s[1])] = (prob, out)
    for b in range(bt.B):
        if need_ctil:
            prob, out = res[(b, "ctil")]
            if isinstance(out, Exception):
                plans.ctil_arcs.append(None)
                plans.ctil_duals.append(None)
                plans.ctil_error.append(out)
            else:
                coupling, duals, _ = out
                plans.ctil_arcs.append((prob.src_index[coupling.row], prob.dst_index[coupling.col],
                                        coupling.mass))
                plans.ctil_duals.append((duals.g, prob.dst_index))
                plans.ctil_error.append(None)
        if need_cbar:
            prob, out = res[(b, "cbar")]
            plans.cbar_value.append(out if isinstance(out, Exception) else out[2])
        if need_cmin:
            prob, out = res[(b, "cmin")]
            plans.cmin_value.append(out if isinstance(out, Exception) else out[2])
    job.cbar_host = None
    return plans


def solve_jobs(jobs, lp_threads: int = 0):
    """Solve the LPs of several jobs as ONE host batch (one thread pool, warm
    chains kept inside each job); returns the plans of every job."""
    problems, warm, spans = [], [], []
    for job in jobs:
        base = len(problems)
        problems.extend(job.problems)
        warm.extend(w if w < 0 else w + base for w in job.warm)
        spans.append((base, len(problems)))
    t = time.perf_counter()
    solved = solve_transport_many(problems, threads=lp_threads, warm_from=warm, slack=False)
    dt = time.perf_counter() - t
    out = []
    for job, (lo, hi) in zip(jobs, spans):
        job.plans.solve_seconds = dt
        out.append(solved[lo:hi])
    return out


def prepare_coarse(bt: _Batch, methods, lp_threads: int = 0) -> CoarsePlans:
    """SumPool + C-bar on the device, then every coarse LP the methods need."""
    t0 = time.perf_counter()
    job = coarse_problems(bt, methods)
    solved = solve_jobs([job], lp_threads)[0]
    plans = assemble_plans(bt, job, solved)
    plans.lp_seconds = time.perf_counter() - t0 - plans.cbar_seconds
    return plans


class _Worker(threading.Thread):
    """Runs one native LP batch off the main thread (the ctypes call releases
    the GIL), so the device work of the orchestrator overlaps it."""

    def __init__(self, fn, *args, **kw):
        super().__init__(daemon=True)
        self.fn, self.args, self.kw = fn, args, kw
        self.result, self.error = None, None

    def run(self):
        try:
            self.result = self.fn(*self.args, **self.kw)
        except BaseException as exc:  # re-raised on the main thread
            self.error = exc

    def get(self):
        self.join()
        if self.error is not None:
            raise self.error
        return self.result


def _pipeline(batches, methods, lp_threads, device_fn, timings=None):
    """Coarse LPs of several batches overlapped with their device work.

    All LPs run as ONE native batch on the host pool, one chain per pair:
    C-tilde (the reference's pivot path; needs only the coarse masses), then
    C-bar and C-min warm-started from the previous optimal basis of the chain.
    The C-bar jobs are held until the device has computed C-bar and copied it
    into their page-locked cost buffers; meanwhile the C-tilde jobs already
    run.  As soon as every C-tilde job of a (kappa, p) batch has finished,
    ``device_fn(i, plans_i)`` runs that batch's device stages (upscaling, IPF,
    c-transforms) while the pool works on the remaining chains.  Values,
    supports and duals are those of the serial order (same LPs, same starts).
    Pairs whose coarse supports are partial get their C-bar LP from a dense
    sub-matrix, built after the batch.  Returns (plans, device results).
    """
    need_ctil = "primal_upscaling" in methods or "dual_upscaling" in methods
    need_cbar = "weighted_cost" in methods
    need_cmin = "min_cost" in methods
    order = sorted(range(len(batches)), key=lambda i: -batches[i].n)  # big LPs first
    t0 = time.perf_counter()
    masses = {i: (to_host(batches[i].mu_c), to_host(batches[i].nu_c)) for i in order}
    plans = {i: CoarsePlans(n=batches[i].n) for i in order}
    pinned = {}

    def build(i, b, cost):
        try:
            return build_transport_problem(masses[i][0][b], masses[i][1][b], cost)
        except GridotError as exc:
            return exc

    probs, warm, hold, slot = [], [], [], {}  # slot[(i, b, kind)] = job index or exception
    late = []  # (i, b): C-bar LPs that need the C-bar values to build (partial supports)
    for i in order:
        bt = batches[i]
        ctil = centre_cost_table(bt.pdims, bt.kappa, bt.p) if need_ctil else None
        cmin = min_cost_table(bt.pdims, bt.kappa, bt.p) if need_cmin else None
        if need_cbar:
            # page-locked C-bar for the host LPs: owned by this call (torch's
            # caching host allocator makes the allocation cheap), released
            # when the call returns, so concurrent calls never share it
            pinned[i] = pinned_empty((bt.B, bt.n, bt.n))
        for b in range(bt.B):
            full = bool((masses[i][0][b] > 0).all() and (masses[i][1][b] > 0).all())
            prev = -1
            first = None  # full supports: the chain's problems share masses and supports
            for kind in ("ctil", "cbar", "cmin"):
                if kind == "ctil" and not need_ctil or kind == "cmin" and not need_cmin:
                    continue
                if kind == "cbar":
                    if not need_cbar:
                        continue
                    if not full:
                        late.append((i, b))
                        continue
                    cost = pinned[i][1][b]  # values arrive before release
                else:
                    cost = ctil if kind == "ctil" else cmin
                if full and first is not None:
                    pr = TransportProblem(first.supply, first.demand, cost, first.src_index,
                                          first.dst_index)
                else:
                    pr = build(i, b, cost)
                    if full and not isinstance(pr, Exception):
                        first = pr
                if isinstance(pr, Exception):
                    slot[(i, b, kind)] = pr
                    continue
                q = len(probs)
                probs.append(pr)
                warm.append(prev)
                if kind == "cbar":
                    hold.append(q)
                slot[(i, b, kind)] = q
                prev = q
    batch = LPBatch(probs, warm_from=warm, hold=hold)
    worker = _Worker(batch.run, lp_threads)
    worker.start()
    t1 = time.perf_counter()
    # C-bar on the device, into the page-locked cost buffers, then release
    try:
        for i in order:
            if not need_cbar:
                break
            vals, _ = _cbar(batches[i], cbar_parent(batches[i], [batches[j] for j in order]))
            pinned[i][0].copy_(vals, non_blocking=True)
            torch().cuda.current_stream(vals.device).synchronize()
            qs = [slot[(i, b, "cbar")] for b in range(batches[i].B)
                  if isinstance(slot.get((i, b, "cbar")), int)]
            batch.release(qs)
    except BaseException:
        batch.release(hold)  # never leave the pool waiting; the error propagates
        worker.join()
        raise
    t2 = time.perf_counter()

    def ctil_jobs(i):
        return [slot[(i, b, "ctil")] for b in range(batches[i].B)
                if isinstance(slot.get((i, b, "ctil")), int)]

    def assemble_ctil(i):
        pl = plans[i]
        for b in range(batches[i].B):
            q = slot.get((i, b, "ctil"))
            out = q if isinstance(q, Exception) else batch.result(q)
            if isinstance(out, Exception):
                pl.ctil_arcs.append(None)
                pl.ctil_duals.append(None)
                pl.ctil_error.append(out)
            else:
                pr = probs[q]
                coupling, duals, _ = out
                pl.ctil_arcs.append((pr.src_index[coupling.row], pr.dst_index[coupling.col],
                                     coupling.mass))
                pl.ctil_duals.append((duals.g, pr.dst_index))
                pl.ctil_error.append(None)

    # device stages of each batch as soon as its C-tilde LPs are done; on an
    # error the native batch is drained first (it reads the pinned buffers)
    dev, pending, t_dev = {}, list(order), 0.0
    try:
        while pending:
            ready_i = [i for i in pending if all(batch.finished(q) for q in ctil_jobs(i))]
            if not ready_i:
                if not worker.is_alive():
                    worker.get()  # surfaces a native failure
                    ready_i = list(pending)
                else:
                    time.sleep(0.0005)
                    continue
            for i in ready_i:
                pending.remove(i)
                if need_ctil:
                    assemble_ctil(i)
                td = time.perf_counter()
                dev[i] = device_fn(i, plans[i])
                t_dev += time.perf_counter() - td
    except BaseException:
        worker.join()
        raise
    t3 = time.perf_counter()
    # C-bar / C-min values as their jobs finish, while the pool runs the rest
    values = {}
    waiting = [(key, q) for key, q in slot.items()
               if key[2] in ("cbar", "cmin") and isinstance(q, int)]
    while waiting:
        still = []
        for key, q in waiting:
            if batch.finished(q):
                values[key] = batch.value(q)
            else:
                still.append((key, q))
        waiting = still
        if waiting:
            if not worker.is_alive():
                break
            time.sleep(0.0005)
    worker.get()
    for key, q in waiting:  # finished as the worker exited
        values[key] = batch.value(q)
    t4 = time.perf_counter()
    # partial-support C-bar LPs (dense sub-matrices of the copied C-bar)
    if late:
        lp_probs, lp_keys = [], []
        for i, b in late:
            pr = build(i, b, pinned[i][1][b])
            if isinstance(pr, Exception):
                slot[(i, b, "cbar")] = pr
            else:
                lp_keys.append((i, b))
                lp_probs.append(pr)
        for (i, b), out in zip(lp_keys, solve_transport_many(lp_probs, threads=lp_threads,
                                                             slack=False)):
            slot[(i, b, "cbar")] = out if isinstance(out, Exception) else ("late", out)
    for i in order:
        for kind, dst in (("cbar", plans[i].cbar_value), ("cmin", plans[i].cmin_value)):
            if kind == "cbar" and not need_cbar or kind == "cmin" and not need_cmin:
                continue
            for b in range(batches[i].B):
                q = slot[(i, b, kind)]
                if isinstance(q, tuple):
                    v = q[1]
                    v = v if isinstance(v, Exception) else v[2]
                elif isinstance(q, Exception):
                    v = q
                else:
                    v = values[(i, b, kind)]
                dst.append(v)
    t5 = time.perf_counter()
    for i in order:
        plans[i].lp_seconds = t4 - t0
        plans[i].solve_seconds = t4 - t1
        plans[i].cbar_seconds = t2 - t1
    if timings is not None:
        for key, val in (("lp_build", t1 - t0), ("cbar", t2 - t1), ("device_overlapped", t_dev),
                         ("lp_tail_wait", t4 - t3), ("lp_late_and_values", t5 - t4)):
            timings[key] = timings.get(key, 0.0) + val
    return plans, dev


# ---------------------------------------------------------------------------
# stage 2: device stages that consume the coarse plans
# ---------------------------------------------------------------------------


def _arc_arrays(bt: _Batch, plans: CoarsePlans):
    """Per-pair CSR (by coarse row) and CSC (by coarse col) arc lists."""
    n = bt.n
    row_ptr = np.zeros((bt.B, n + 1), np.int32)
    col_ptr = np.zeros((bt.B, n + 1), np.int32)
    rcol, rmass, crow, cmass = [], [], [], []
    off = [0]
    for b in range(bt.B):
        arcs = plans.ctil_arcs[b]
        if arcs is None:
            off.append(off[-1])
            continue
        r, c, m = (np.asarray(x) for x in arcs)
        o = np.lexsort((c, r))
        rcol.append(c[o].astype(np.int32))
        rmass.append(m[o])
        row_ptr[b, 1:] = np.cumsum(np.bincount(r, minlength=n))
        o = np.lexsort((r, c))
        crow.append(r[o].astype(np.int32))
        cmass.append(m[o])
        col_ptr[b, 1:] = np.cumsum(np.bincount(c, minlength=n))
        off.append(off[-1] + len(r))
    cat = lambda xs, dt: np.concatenate(xs).astype(dt) if xs else np.zeros(1, dt)  # noqa: E731
    return (np.array(off, np.int64), row_ptr, cat(rcol, np.int32), cat(rmass, np.float64),
            col_ptr, cat(crow, np.int32), cat(cmass, np.float64))


class DevicePlans:
    """Coarse plans uploaded once: arc CSR/CSC lists, duals, lattice axes, scratch."""

    def __init__(self, bt: _Batch, plans: CoarsePlans, paired=None, xi=None):
        t = bt.t
        self.plans = plans
        if paired is None:
            paired = _uniform_paired(bt.kappa, bt.d)
        self.uniform = bool(np.all(paired == paired.flat[0]))
        self.W = to_dev(np.ascontiguousarray(paired))
        self.xi = to_dev(np.full(bt.B, -1.0 if xi is None else float(xi)))
        self.has_arcs = bool(plans.ctil_arcs)
        if self.has_arcs:
            (self.arc_off, self.row_ptr, self.rcol, self.rmass, self.col_ptr, self.crow,
             self.cmass) = (to_dev(a) for a in _arc_arrays(bt, plans))
            n, B = bt.n, bt.B
            g = np.zeros((B, n))
            dst = np.zeros((B, n), np.int32)
            slen = np.zeros(B, np.int32)
            for b in range(B):
                if plans.ctil_duals[b] is None:
                    continue
                gb, di = plans.ctil_duals[b]
                g[b, :len(gb)] = gb
                dst[b, :len(di)] = di
                slen[b] = len(di)
            self.g, self.dst, self.slen = to_dev(g), to_dev(dst), to_dev(slen)
        centres = coarsen_grid(GridSpec(bt.dims), CoarseningSpec(bt.kappa))
        self.axes = to_dev(np.concatenate([np.unique(centres[:, a]) for a in range(bt.d)]))
        nbytes = N.lib().gdt_primal_scratch_bytes(bt.B, bt.d, N.i64s(bt.pdims), bt.kappa,
                                                  int(self.uniform))
        self.primal_scratch = t.empty(max(nbytes // 8, 1), dtype=t.float64, device=bt.dev)
        self.dt = 1 if bt.precision == "fp32" else 0
        if self.dt == 1 and bt.dims[0] % 8 != 0 and bt.p != 2.0:
            self.dt = 0  # the fp32 brute kernel tiles axis 0 by 8
        self.ct_bytes = N.lib().gdt_ctransform_scratch_bytes(bt.B, bt.d, N.i64s(bt.dims), bt.p,
                                                             self.dt)
        self.ct_scratch = t.empty(max(self.ct_bytes, 8), dtype=t.uint8, device=bt.dev)
        Nf = int(np.prod(bt.dims))
        tdt = t.float32 if self.dt else t.float64
        self.f_ext = t.empty((bt.B, bt.n), dtype=t.float64, device=bt.dev)
        self.f_hat = t.empty((bt.B, Nf), dtype=t.float64, device=bt.dev)
        self.gf = t.empty((bt.B, Nf), dtype=tdt, device=bt.dev)
        self.ff = t.empty((bt.B, Nf), dtype=tdt, device=bt.dev)
        self.dots = t.empty((2, bt.B), dtype=t.float64, device=bt.dev)
        self.prim_out = t.empty((bt.B, 8), dtype=t.float64, device=bt.dev)
        self.prim_status = t.empty(bt.B, dtype=t.int32, device=bt.dev)


_GRID_TABLES = {}
_GRID_LOCK = threading.Lock()


def _grid_tables(pdims, kappa, p):
    """Device copies of the padded grid's tv_weights (the reference's own
    formula, measures.py:289-296) and its cell -> coarse block map, cached per
    (device, grid, kappa, p)."""
    key = (torch().cuda.current_device(), tuple(pdims), int(kappa), float(p))
    with _GRID_LOCK:
        hit = _GRID_TABLES.get(key)
        if hit is None:
            grid = GridSpec(tuple(pdims))
            hit = (to_dev(tv_weights(grid, float(p))),
                   to_dev(block_index_map(grid, CoarseningSpec(int(kappa))).astype(np.int32)))
            _GRID_TABLES[key] = hit
    return hit


def launch_primal(bt: _Batch, dp: DevicePlans, max_iter):
    # fp32 mode with C-bar at hand (the weighted-cost bound computed it): the
    # coarse-level primal stage, priced by C-bar (primal.cu primal_coarse_kernel)
    cbar = bt.cbar_dev if (bt.mode == 1 and dp.uniform) else None
    # the padded grid's tv_weights (the reference's formula, host-computed) and
    # cell -> block map: the coarse-level stage needs both, the fine-level
    # kernels read the weights instead of recomputing them per cell
    tv_w, bmap = _grid_tables(bt.pdims, bt.kappa, bt.p)
    N.check(N.lib().gdt_primal_upscale(
        N.ptr(bt.mu_pad), N.ptr(bt.nu_pad), N.ptr(bt.mu_c), N.ptr(bt.nu_c), N.ptr(bt.stats),
        N.ptr(cbar), N.ptr(tv_w), N.ptr(bmap), N.ptr(dp.arc_off), N.ptr(dp.row_ptr),
        N.ptr(dp.rcol),
        N.ptr(dp.rmass), N.ptr(dp.col_ptr), N.ptr(dp.crow), N.ptr(dp.cmass), N.ptr(dp.W),
        int(dp.uniform), N.ptr(dp.xi), int(max_iter), bt.p, bt.B, bt.d, N.i64s(bt.pdims),
        bt.kappa, N.ptr(bt.table_dev), bt.max_sq, bt.mode, N.ptr(dp.prim_out),
        N.ptr(dp.prim_status),
        N.ptr(dp.primal_scratch), stream()), "gdt_primal_upscale")
    return dp.prim_out, dp.prim_status


def launch_dual_prep(bt: _Batch, dp: DevicePlans, method: str = "multilinear"):
    N.check(N.lib().gdt_coarse_ctransform(N.ptr(dp.g), N.ptr(dp.dst), N.ptr(dp.slen),
                                          N.ptr(bt.ctil_dev), bt.n, bt.B, N.ptr(dp.f_ext),
                                          stream()), "gdt_coarse_ctransform")
    N.check(N.lib().gdt_interpolate(N.ptr(dp.f_ext), N.ptr(dp.f_hat), bt.B, bt.d,
                                    N.i64s(bt.dims), N.i64s(bt.cdims), N.ptr(dp.axes),
                                    1 if method == "nearest" else 0, stream()), "gdt_interpolate")


def launch_ctransform(bt: _Batch, dp: DevicePlans, which: int):
    """which = 0: g = T f_hat (dot with nu); 1: f = T g (dot with mu)."""
    src, dst, mass, dot, in_dt = ((dp.f_hat, dp.gf, bt.nu, dp.dots[1], 0) if which == 0 else
                                  (dp.gf, dp.ff, bt.mu, dp.dots[0], dp.dt))
    N.check(N.lib().gdt_ctransform_grid(N.ptr(src), N.ptr(dst), bt.B, bt.d, N.i64s(bt.dims),
                                        bt.p, dp.dt, in_dt, N.ptr(bt.table_dev), bt.max_sq,
                                        N.ptr(mass), N.ptr(dot), N.ptr(dp.ct_scratch),
                                        dp.ct_bytes, stream()), "gdt_ctransform_grid")


def ctransform_pair(f_hat, mu, nu, dims, p, precision, table_dev=None, max_sq=0):
    """g = T f_hat, f = T g on the fine grid; returns (f, g, dots [f.mu, g.nu])."""
    t = torch()
    B, Nf = f_hat.shape
    dt = 1 if precision == "fp32" else 0
    if p != 2.0 and table_dev is None:
        max_sq = max_sq_of(dims)
        table_dev = to_dev(cost_table(max_sq, float(p)))
    if dt == 1 and dims[0] % 8 != 0 and p != 2.0:
        dt = 0
    tdt = t.float32 if dt else t.float64
    nbytes = N.lib().gdt_ctransform_scratch_bytes(B, len(dims), N.i64s(dims), float(p), dt)
    scratch = t.empty(max(nbytes, 8), dtype=t.uint8, device=f_hat.device)
    g = t.empty((B, Nf), dtype=tdt, device=f_hat.device)
    f = t.empty((B, Nf), dtype=tdt, device=f_hat.device)
    dots = t.empty((2, B), dtype=t.float64, device=f_hat.device)
    N.check(N.lib().gdt_ctransform_grid(N.ptr(f_hat), N.ptr(g), B, len(dims), N.i64s(dims),
                                        float(p), dt, 0, N.ptr(table_dev), max_sq, N.ptr(nu),
                                        N.ptr(dots[1]), N.ptr(scratch), nbytes, stream()),
            "gdt_ctransform_grid(target)")
    N.check(N.lib().gdt_ctransform_grid(N.ptr(g), N.ptr(f), B, len(dims), N.i64s(dims),
                                        float(p), dt, dt, N.ptr(table_dev), max_sq, N.ptr(mu),
                                        N.ptr(dots[0]), N.ptr(scratch), nbytes, stream()),
            "gdt_ctransform_grid(source)")
    return f, g, dots


def gpu_stages(bt: _Batch, dp: DevicePlans, methods, max_iter=10_000, dual_method="multilinear"):
    """Device work downstream of the LPs (results stay on the device)."""
    res = {}
    if "primal_upscaling" in methods:
        res["primal"] = launch_primal(bt, dp, max_iter)
    if "dual_upscaling" in methods:
        launch_dual_prep(bt, dp, dual_method)
        launch_ctransform(bt, dp, 0)
        launch_ctransform(bt, dp, 1)
        res["dual"] = dp.dots
    return res


# ---------------------------------------------------------------------------
# host finishing (reference arithmetic) and the ring fallback
# ---------------------------------------------------------------------------


def _ring_fallback(bt: _Batch, b: int, plans: CoarsePlans, xi, max_iter):
    """One-ring respread + generic CSR IPF on the device (quantized.py:335-344)."""
    from .sinkhorn import ipf_fit_device
    from .quantized import _one_ring_spread_host

    rows, cols, mass = plans.ctil_arcs[b]
    fr, fc, fm = _one_ring_spread_host(rows, cols, mass, bt.cdims, bt.pdims, bt.kappa)
    mu_p = to_host(bt.mu_pad[b])
    nu_p = to_host(bt.nu_pad[b])
    return ipf_fit_device(fr, fc, fm, mu_p, nu_p, bt.pdims, bt.p, xi, max_iter, bt.table_dev,
                          bt.max_sq)


def _primal_report(p, price, tmu, tnu, gap, iters, conv, n, wall):
    transport = float(price) ** (1.0 / p)
    dmu = 2.0 ** (1.0 - 1.0 / p) * float(tmu) ** (1.0 / p)
    dnu = 2.0 ** (1.0 - 1.0 / p) * float(tnu) ** (1.0 / p)
    value = transport + dmu + dnu
    return BoundReport("primal_upscaling", value, value,
                       {"transport": transport, "delta_mu": dmu, "delta_nu": dnu,
                        "marginal_gap": float(gap), "converged": float(conv)},
                       wall, int(iters), n)


def _check_args(precision, methods):
    if precision not in PRECISIONS:
        raise ValueError(f"precision must be one of {PRECISIONS}")
    for m in methods:
        if m not in QUANT_METHODS:
            raise ValueError(f"unknown method {m!r}")


def _device_masses(mus, nus, dims):
    device()
    mu = to_dev(mus)
    nu = to_dev(nus)
    if mu.dim() == 1:
        mu, nu = mu[None, :], nu[None, :]
    if mu.shape != nu.shape or mu.shape[1] != int(np.prod(dims)):
        raise DimensionMismatchError(f"masses {tuple(mu.shape)} do not match dims {dims}")
    return mu, nu


def _kernel_pairs(bt: _Batch, kernel):
    if kernel is None:
        return None
    if kernel.kappa != bt.kappa or kernel.ndim != bt.d:
        raise DimensionMismatchError(
            f"kernel is ({kernel.kappa}, {kernel.ndim}), expected ({bt.kappa}, {bt.d})")
    return kernel.paired()


def _run_device(bt: _Batch, plans: CoarsePlans, paired, xi, max_iter, methods, dual_method):
    dp = DevicePlans(bt, plans, paired, xi)
    t_dp = time.perf_counter()
    res = gpu_stages(bt, dp, methods, max_iter, dual_method)
    prim = None
    if "primal" in res:
        out, status = res["primal"]
        prim = (to_host(out), to_host(status))
    dual = to_host(res["dual"]) if "dual" in res else None
    return prim, dual, t_dp


def _reports(bt: _Batch, plans: CoarsePlans, prim, dual, methods, xi, max_iter, wall,
             return_exceptions, timings):
    reports = []
    for b in range(bt.B):
        rep = {}
        if "weighted_cost" in methods:
            v = plans.cbar_value[b]
            if isinstance(v, Exception):
                rep["weighted_cost"] = v
            else:
                val = v ** (1.0 / bt.p)
                rep["weighted_cost"] = BoundReport("weighted_cost", val, val, {"transport": val},
                                                   wall, None, bt.n)
        if "min_cost" in methods:
            v = plans.cmin_value[b]
            if isinstance(v, Exception):
                rep["min_cost"] = v
            else:
                raw = signed_root(v, bt.p)
                rep["min_cost"] = BoundReport("min_cost", max(0.0, raw), raw, {"transport": raw},
                                              wall, None, bt.n)
        err = plans.ctil_error[b] if plans.ctil_error else None
        if "primal_upscaling" in methods:
            if err is not None:
                rep["primal_upscaling"] = err
            else:
                o, st = prim[0][b], int(prim[1][b])
                try:
                    if st in (1, 2):
                        if timings is not None:
                            timings["ring_fallbacks"] = timings.get("ring_fallbacks", 0) + 1
                        o = _ring_fallback(bt, b, plans, xi, max_iter)
                        st = 0
                    if st == 3:
                        raise NumericOverflowError("scaling vector left [1e-100, 1e100]")
                    rep["primal_upscaling"] = _primal_report(bt.p, o[0], o[1], o[2], o[3], o[4],
                                                             o[5], bt.n, wall)
                except GridotError as exc:
                    rep["primal_upscaling"] = exc
        if "dual_upscaling" in methods:
            if err is not None:
                rep["dual_upscaling"] = err
            else:
                dv = float(dual[0][b] + dual[1][b])
                raw = signed_root(dv, bt.p)
                rep["dual_upscaling"] = BoundReport("dual_upscaling", max(0.0, raw), raw,
                                                    {"dual_value": dv}, wall, None, bt.n)
        if not return_exceptions:
            for v in rep.values():
                if isinstance(v, Exception):
                    raise v
        reports.append(rep)
    return reports


# page-locked C-bar held for the host LPs of one pipeline run; larger batches
# are processed in consecutive chunks of pairs (each a full pipeline run)
PINNED_BUDGET_BYTES = 4 << 30


def _chunks(B, dims, combos, methods, max_chunk_pairs):
    """[lo, hi) pair ranges: each keeps the C-bar of all combinations under
    PINNED_BUDGET_BYTES (pinned host) unless max_chunk_pairs says otherwise."""
    if max_chunk_pairs is None:
        per_pair = 0
        if "weighted_cost" in methods:
            for k, _ in combos:
                n = int(np.prod([-(-x // int(k)) for x in dims]))
                per_pair += 8 * n * n
        max_chunk_pairs = max(1, PINNED_BUDGET_BYTES // max(per_pair, 1))
    step = max(1, int(max_chunk_pairs))
    return [(lo, min(B, lo + step)) for lo in range(0, B, step)] or [(0, 0)]


def _export_plans(plans_out, key, plans: CoarsePlans):
    if plans_out is None:
        return
    dst = plans_out.setdefault(key, [])
    for b in range(len(plans.ctil_arcs)):
        arcs, duals = plans.ctil_arcs[b], plans.ctil_duals[b]
        dst.append(None if arcs is None else (arcs[0], arcs[1], arcs[2], duals[0], duals[1]))


def quantized_bounds(mus, nus, dims, kappa, p, *, precision="fp64", xi=None, max_iter=10_000,
                     kernel=None, methods=QUANT_METHODS, dual_method="multilinear",
                     lp_threads=0, return_exceptions=True, timings=None, max_chunk_pairs=None,
                     plans_out=None):
    """All requested quantization bounds for a batch of pairs on one grid.

    mus, nus: [B, prod(dims)] float64 (numpy, pinned or device tensors).
    Returns a list (one per pair) of {method: BoundReport | exception}.
    Pairs are processed in chunks (``max_chunk_pairs``, default: as many as
    keep the page-locked C-bar under PINNED_BUDGET_BYTES); ``plans_out``
    (a dict) receives, under key (kappa, p), each pair's C-tilde plan
    (full coarse rows, cols, masses, dual g, its support index) or None.
    """
    _check_args(precision, methods)
    t_start = time.perf_counter()
    mu, nu = _device_masses(mus, nus, dims)
    reports = []
    for lo, hi in _chunks(mu.shape[0], dims, [(kappa, p)], methods, max_chunk_pairs):
        tc = time.perf_counter()
        bt = _Batch(mu[lo:hi], nu[lo:hi], dims, kappa, p, precision)
        paired = _kernel_pairs(bt, kernel)
        t0 = time.perf_counter()
        plans, dev = _pipeline([bt], methods, lp_threads,
                               lambda i, pl: _run_device(bt, pl, paired, xi, max_iter, methods,
                                                         dual_method), timings)
        plans = plans[0]
        prim, dual, _ = dev[0]
        t2 = time.perf_counter()
        if timings is not None:
            timings["prepare"] = timings.get("prepare", 0.0) + t0 - tc
            timings["coarse_and_gpu"] = timings.get("coarse_and_gpu", 0.0) + t2 - t0
        wall = (t2 - (t_start if lo == 0 else tc)) / max(bt.B, 1)
        _export_plans(plans_out, (int(kappa), float(p)), plans)
        reports += _reports(bt, plans, prim, dual, methods, xi, max_iter, wall,
                            return_exceptions, timings)
        if timings is not None:
            timings["finish"] = timings.get("finish", 0.0) + time.perf_counter() - t2
    return reports


def quantized_bounds_many(mus, nus, dims, combos, *, precision="fp64", xi=None,
                          max_iter=10_000, methods=QUANT_METHODS, dual_method="multilinear",
                          lp_threads=0, return_exceptions=True, timings=None,
                          max_chunk_pairs=None, plans_out=None):
    """:func:`quantized_bounds` for several (kappa, p) combinations of the same
    batch at once: the masses are uploaded once, and the coarse LPs of ALL
    combinations run as one host batch on one thread pool (the expensive
    combinations' LPs first), which keeps every core busy where one batch per
    combination leaves the tail of each wave idle.  Results and their values
    are those of one ``quantized_bounds`` call per combination (the same LPs,
    pivot paths and device kernels), with one exception in fp32 mode: for
    p != 2, C-bar at a pooling factor that is a multiple of another requested
    one on the same padded grid is pooled from that finer C-bar (the numerator
    is additive over nested blocks) instead of a second pass over the fine
    cells -- equal to rounding, inside the fp32 contract; ``BoundReport.wall_time`` is the whole
    call's wall time per pair and combination.  ``max_chunk_pairs`` and
    ``plans_out`` as in :func:`quantized_bounds`.

    Returns {(kappa, p): [per-pair {method: BoundReport | exception}]}.
    """
    _check_args(precision, methods)
    t_start = time.perf_counter()
    mu, nu = _device_masses(mus, nus, dims)
    combos = [(int(k), float(p)) for k, p in combos]
    out = {key: [] for key in combos}
    for lo, hi in _chunks(mu.shape[0], dims, combos, methods, max_chunk_pairs):
        tc = time.perf_counter()
        batches = [_Batch(mu[lo:hi], nu[lo:hi], dims, k, p, precision) for k, p in combos]
        t0 = time.perf_counter()
        plans, dev = _pipeline(batches, methods, lp_threads,
                               lambda i, pl: _run_device(batches[i], pl, None, xi, max_iter,
                                                         methods, dual_method), timings)
        t3 = time.perf_counter()
        nb = max(hi - lo, 1)
        wall = (t3 - (t_start if lo == 0 else tc)) / nb / max(len(combos), 1)
        for i, key in enumerate(combos):
            prim, dual, _ = dev[i]
            _export_plans(plans_out, key, plans[i])
            out[key] += _reports(batches[i], plans[i], prim, dual, methods, xi, max_iter, wall,
                                 return_exceptions, timings)
        if timings is not None:
            timings["prepare"] = timings.get("prepare", 0.0) + t0 - tc
            timings["coarse_and_gpu"] = timings.get("coarse_and_gpu", 0.0) + t3 - t0
            timings["finish"] = timings.get("finish", 0.0) + time.perf_counter() - t3
    return out


def make_batch(mus, nus, dims, kappa, p, precision="fp64"):
    """Device-resident batch (for benchmarks and staged use)."""
    device()
    return _Batch(to_dev(mus), to_dev(nus), dims, kappa, p, precision)


ZeroDenominatorError = ZeroDenominatorError  # re-export for callers of the engine
