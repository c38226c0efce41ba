"""Iterative proportional fitting and the entropic bounds on the device
(reference: sinkhorn.py).

``ipf_fit`` is the reference's generic entry point: any dense / scipy-sparse
kernel (or a MatrixLinearOperator wrapping one) is turned into a canonical
CSR + CSC pair and fitted by ``gdt_ipf_csr`` in libgridot_b200.so, whose row
and column sums follow scipy's CSR/CSC mat-vec order.  The primal bound uses
the specialised block-sparse kernel instead (engine.py / primal.cu); this
generic path serves explicit kernels and the one-ring fallback.

The entropic-regularisation bounds (``reg_lower_bound`` / ``reg_upper_bound``,
sinkhorn.py:150-299) run the alternating scaling on the dense support-
restricted Gibbs kernel in HBM with the log-domain restart of the reference
(``gdt_entropic_fit``, entropic.cu) and price the fitted plan on the device
(``gdt_entropic_plan``); the dual dot products and the TV corrections are the
reference's host/device formulas.
"""

from __future__ import annotations

import logging
import time
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import _native as N
from .device import device, stream, to_dev, to_host, torch
from .errors import (DimensionMismatchError, GridMismatchError, KernelSizeError,
                     NumericOverflowError, UnbalancedError, ZeroDenominatorError)
from .reports import BoundReport, signed_root

__all__ = ["IpfState", "ipf_fit", "ipf_fit_device", "SCALE_FLOOR", "SCALE_CEIL",
           "MAX_KERNEL_CELLS", "RegularizationParams", "reg_lower_bound", "reg_upper_bound"]

logger = logging.getLogger(__name__)

# dense Gibbs kernels are materialised only up to this many cells (sinkhorn.py:38)
MAX_KERNEL_CELLS = 1 << 16
SCALE_FLOOR = 1e-100
SCALE_CEIL = 1e100


@dataclass(frozen=True)
class RegularizationParams:
    """Knobs of the entropic bounds (sinkhorn.py:46-69): ``epsilon`` in cost
    units, the L1 marginal-drift threshold ``xi`` (None: 1e-9 times the
    number of support points of the pair) and the sweep cap."""

    epsilon: float
    xi: float | None = None
    max_iter: int = 10_000

    def __post_init__(self):
        if not self.epsilon > 0.0:
            raise ValueError(f"epsilon must be positive, got {self.epsilon}")
        if self.xi is not None and not self.xi > 0.0:
            raise ValueError(f"xi must be positive, got {self.xi}")
        if self.max_iter < 1:
            raise ValueError(f"max_iter must be at least 1, got {self.max_iter}")

    def resolve_xi(self, support_points: int) -> float:
        return self.xi if self.xi is not None else 1e-9 * support_points


@dataclass
class IpfState:
    """Final scaling vectors and convergence record (sinkhorn.py:72-85)."""

    a: np.ndarray
    b: np.ndarray
    iterations: int
    marginal_gap: float
    converged: bool


def _as_csr(kernel_apply) -> sp.csr_array:
    k = kernel_apply
    if hasattr(k, "A") and not sp.issparse(k) and not isinstance(k, np.ndarray):
        k = k.A  # scipy MatrixLinearOperator
    if sp.issparse(k):
        mat = sp.csr_array(k, dtype=np.float64)
    elif isinstance(k, np.ndarray):
        mat = sp.csr_array(np.asarray(k, dtype=np.float64))
    else:
        raise TypeError("ipf_fit needs a dense array, a scipy sparse matrix or a "
                        "MatrixLinearOperator; opaque operators cannot run on the device")
    mat.sum_duplicates()
    mat.sort_indices()
    return mat


def _status_raise(st: int):
    if st == 1:
        raise ZeroDenominatorError("kernel row support cannot reach a positive source marginal")
    if st == 2:
        raise ZeroDenominatorError("kernel column support cannot reach a positive target marginal")
    if st == 3:
        raise NumericOverflowError(f"scaling vector left [{SCALE_FLOOR:g}, {SCALE_CEIL:g}]")


def _run_csr(mat: sp.csr_array, mu, nu, xi, max_iter):
    t = torch()
    csc = mat.tocsc()
    csc.sort_indices()
    nr, nc = mat.shape
    indptr = to_dev(mat.indptr.astype(np.int64))
    indices = to_dev(mat.indices.astype(np.int32))
    data = to_dev(mat.data.astype(np.float64))
    tindptr = to_dev(csc.indptr.astype(np.int64))
    tindices = to_dev(csc.indices.astype(np.int32))
    tdata = to_dev(csc.data.astype(np.float64))
    mu_d, nu_d = to_dev(np.asarray(mu, np.float64)), to_dev(np.asarray(nu, np.float64))
    a = t.empty(nr, dtype=t.float64, device=mu_d.device)
    kb = t.empty(nr, dtype=t.float64, device=mu_d.device)
    b = t.empty(nc, dtype=t.float64, device=mu_d.device)
    kta = t.empty(nc, dtype=t.float64, device=mu_d.device)
    info = t.empty(4, dtype=t.float64, device=mu_d.device)
    status = t.empty(1, dtype=t.int32, device=mu_d.device)
    N.check(N.lib().gdt_ipf_csr(N.ptr(indptr), N.ptr(indices), N.ptr(data), N.ptr(tindptr),
                                N.ptr(tindices), N.ptr(tdata), N.ptr(mu_d), N.ptr(nu_d), nr, nc,
                                float(xi), int(max_iter), N.ptr(a), N.ptr(b), N.ptr(kb),
                                N.ptr(kta), N.ptr(info), N.ptr(status), stream()), "gdt_ipf_csr")
    _status_raise(int(to_host(status)[0]))
    inf = to_host(info)
    return a, b, kb, kta, int(inf[0]), float(inf[1]), bool(inf[2] != 0.0)


def ipf_fit(kernel_apply, mu, nu, xi: float, max_iter: int = 10_000) -> IpfState:
    """Fit diag(a) K diag(b) to (mu, nu) on the device (sinkhorn.py:101-142)."""
    device()
    mat = _as_csr(kernel_apply)
    if mat.shape != (len(mu), len(nu)):
        raise ValueError(f"kernel shape {mat.shape} does not match marginals")
    a, b, _, _, it, gap, conv = _run_csr(mat, mu, nu, xi, max_iter)
    return IpfState(to_host(a), to_host(b), it, gap, conv)


def ipf_fit_device(rows, cols, mass, mu_pad, nu_pad, pdims, p, xi, max_iter, table_dev,
                   max_sq):
    """Fit + price + TV of an explicit fine coupling on the padded grid.

    Used for the one-ring fallback (quantized.py:322-365).  Returns the raw
    scalars (price, tv_mu, tv_nu, gap, iterations, converged)."""
    t = torch()
    n = int(np.prod(pdims))
    src = np.flatnonzero(mu_pad > 0.0)
    dst = np.flatnonzero(nu_pad > 0.0)
    if xi is None:
        xi = 1e-9 * (src.size + dst.size)
    rpos = np.full(n, -1)
    rpos[src] = np.arange(src.size)
    cpos = np.full(n, -1)
    cpos[dst] = np.arange(dst.size)
    keep = (rpos[rows] >= 0) & (cpos[cols] >= 0)
    fr, fc, fm = rows[keep], cols[keep], mass[keep]
    mat = sp.csr_array((fm, (rpos[fr], cpos[fc])), shape=(src.size, dst.size))
    mat.sum_duplicates()
    mat.sort_indices()
    a, b, kb, kta, it, gap, conv = _run_csr(mat, mu_pad[src], nu_pad[dst], xi, max_iter)
    dev = a.device
    src_d, dst_d = to_dev(src.astype(np.int64)), to_dev(dst.astype(np.int64))
    a_full = t.zeros(n, dtype=t.float64, device=dev)
    b_full = t.zeros(n, dtype=t.float64, device=dev)
    a_full[src_d] = a
    b_full[dst_d] = b
    mu_hat = t.zeros((1, n), dtype=t.float64, device=dev)
    nu_hat = t.zeros((1, n), dtype=t.float64, device=dev)
    mu_hat[0, src_d] = a * kb
    nu_hat[0, dst_d] = b * kta
    price = t.empty(1, dtype=t.float64, device=dev)
    r_d, c_d, m_d = to_dev(fr.astype(np.int64)), to_dev(fc.astype(np.int64)), to_dev(fm)
    N.check(N.lib().gdt_price_coo(N.ptr(r_d), N.ptr(c_d), N.ptr(m_d), len(fr), N.ptr(a_full),
                                  N.ptr(b_full), N.ptr(table_dev), max_sq, float(p), len(pdims),
                                  N.i64s(pdims), N.ptr(price), stream()), "gdt_price_coo")
    tv = t.empty(2, dtype=t.float64, device=dev)
    mu_p, nu_p = to_dev(mu_pad[None, :]), to_dev(nu_pad[None, :])
    for idx, (hat, marg) in enumerate(((mu_hat, mu_p), (nu_hat, nu_p))):
        N.check(N.lib().gdt_weighted_tv_inner(N.ptr(hat), N.ptr(marg), 1, len(pdims),
                                              N.i64s(pdims), float(p), None, N.ptr(tv[idx:]),
                                              stream()), "gdt_weighted_tv_inner")
    pr, tvh = to_host(price), to_host(tv)
    return (float(pr[0]), float(tvh[0]), float(tvh[1]), gap, it, 1.0 if conv else 0.0)


# ---------------------------------------------------------------------------
# entropic bounds (sinkhorn.py:150-299)
# ---------------------------------------------------------------------------


def _prepare_pair(mu, nu, cost):
    """Checks and support restriction of sinkhorn.py:198-223."""
    if mu.grid != nu.grid:
        raise GridMismatchError(f"grids differ: {mu.grid.dims} vs {nu.grid.dims}")
    n = mu.grid.cell_count
    if cost.n_source != n or cost.n_target != n:
        raise DimensionMismatchError(
            f"cost is {cost.n_source}x{cost.n_target} but the grid has {n} cells")
    if n > MAX_KERNEL_CELLS:
        raise KernelSizeError(
            f"dense kernel refused for {n} cells (cap {MAX_KERNEL_CELLS}); "
            "use the quantization bounds at this scale")
    if abs(mu.total_mass - nu.total_mass) > 1e-9:
        raise UnbalancedError(f"total masses differ: {mu.total_mass!r} vs {nu.total_mass!r}")
    src, dst = mu.support, nu.support
    return src, dst, mu.mass[src], nu.mass[dst]


class _EntropicFit:
    """Device buffers of one fitted pair (support coordinates, potentials)."""

    def __init__(self, mu, nu, cost, params):
        self.src, self.dst, self.mu_s, self.nu_s = _prepare_pair(mu, nu, cost)
        self.p, self.eps = float(cost.p), float(params.epsilon)
        self.ns, self.nt = self.src.size, self.dst.size
        self.d = cost.source.shape[1]
        xi = params.resolve_xi(self.ns + self.nt)
        device()
        t = torch()
        self.xs = to_dev(np.ascontiguousarray(cost.source[self.src]))
        self.xt = to_dev(np.ascontiguousarray(cost.target[self.dst]))
        mu_d, nu_d = to_dev(self.mu_s), to_dev(self.nu_s)
        dev = mu_d.device
        nbytes = int(N.lib().gdt_entropic_scratch_bytes(self.ns, self.nt))
        self.scratch = t.empty(nbytes, dtype=t.uint8, device=dev)
        self.f = t.empty(self.ns, dtype=t.float64, device=dev)
        self.g = t.empty(self.nt, dtype=t.float64, device=dev)
        info = t.empty(4, dtype=t.float64, device=dev)
        status = t.empty(1, dtype=t.int32, device=dev)
        N.check(N.lib().gdt_entropic_fit(
            N.ptr(self.xs), N.ptr(self.xt), self.ns, self.nt, self.d, self.p, self.eps,
            N.ptr(mu_d), N.ptr(nu_d), float(xi), int(params.max_iter), N.ptr(self.f),
            N.ptr(self.g), N.ptr(info), N.ptr(status), N.ptr(self.scratch), stream()),
            "gdt_entropic_fit")
        it, gap, conv, logd = to_host(info)
        if logd:
            logger.info("plain scaling failed; restarted in log domain")
        if int(to_host(status)[0]) != 0:
            raise NumericOverflowError("log-domain potentials are not finite")
        self.iterations, self.gap, self.converged = int(it), float(gap), bool(conv)


def reg_lower_bound(mu, nu, cost, params: RegularizationParams) -> BoundReport:
    """Lower bound from the duals of the entropic fit (sinkhorn.py:226-256):
    ``(<f, mu> + <g, nu>)**(1/p)`` with f = eps log a, g = eps log b; a negative
    dual value stays in ``raw_value`` and is clipped to 0 in ``value``."""
    start = time.perf_counter()
    fit = _EntropicFit(mu, nu, cost, params)
    dual_value = float(to_host(fit.f) @ fit.mu_s + to_host(fit.g) @ fit.nu_s)
    raw = signed_root(dual_value, fit.p)
    return BoundReport(
        method="reg_lower", value=max(0.0, raw), raw_value=raw,
        components={"dual_value": dual_value, "marginal_gap": fit.gap,
                    "converged": float(fit.converged)},
        wall_time=time.perf_counter() - start, iterations=fit.iterations)


def reg_upper_bound(mu, nu, cost, params: RegularizationParams) -> BoundReport:
    """Upper bound from the fitted plan plus weighted-TV drift corrections
    (sinkhorn.py:259-299): the plan exp((f + g - C) / eps) is priced on the
    device and its marginals are charged against (mu, nu)."""
    from .measures import GridMeasure, tv_weights, weighted_tv

    start = time.perf_counter()
    fit = _EntropicFit(mu, nu, cost, params)
    t = torch()
    dev = fit.f.device
    mu_hat_s = t.empty(fit.ns, dtype=t.float64, device=dev)
    nu_hat_s = t.empty(fit.nt, dtype=t.float64, device=dev)
    total = t.empty(1, dtype=t.float64, device=dev)
    N.check(N.lib().gdt_entropic_plan(
        N.ptr(fit.xs), N.ptr(fit.xt), fit.ns, fit.nt, fit.d, fit.p, fit.eps, N.ptr(fit.f),
        N.ptr(fit.g), N.ptr(mu_hat_s), N.ptr(nu_hat_s), N.ptr(total), N.ptr(fit.scratch),
        stream()), "gdt_entropic_plan")
    transport = float(to_host(total)[0]) ** (1.0 / fit.p)
    n = mu.grid.cell_count
    mu_hat, nu_hat = np.zeros(n), np.zeros(n)
    mu_hat[fit.src] = to_host(mu_hat_s)
    nu_hat[fit.dst] = to_host(nu_hat_s)
    weights = tv_weights(mu.grid, fit.p)
    delta_mu = weighted_tv(GridMeasure(mu.grid, mu_hat), mu, weights, fit.p)
    delta_nu = weighted_tv(GridMeasure(nu.grid, nu_hat), nu, weights, fit.p)
    value = transport + delta_mu + delta_nu
    return BoundReport(
        method="reg_upper", value=value, raw_value=value,
        components={"transport": transport, "delta_mu": delta_mu, "delta_nu": delta_nu,
                    "marginal_gap": fit.gap, "converged": float(fit.converged)},
        wall_time=time.perf_counter() - start, iterations=fit.iterations)
