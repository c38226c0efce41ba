"""Iterative proportional fitting on the device (reference: sinkhorn.py:72-142).

``ipf_fit`` is the reference's generic entry point: any dense / scipy-sparse
kernel (or a MatrixLinearOperator wrapping one) is turned into a canonical
CSR + CSC pair and fitted by ``gdt_ipf_csr`` in libgridot_b200.so, whose row
and column sums follow scipy's CSR/CSC mat-vec order.  The primal bound uses
the specialised block-sparse kernel instead (engine.py / primal.cu); this
generic path serves explicit kernels and the one-ring fallback.

The entropic-regularisation bounds of sinkhorn.py (reg_lower/upper_bound) are
not on the north-star hot path and are out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import _native as N
from .device import device, stream, to_dev, to_host, torch
from .errors import NumericOverflowError, ZeroDenominatorError

__all__ = ["IpfState", "ipf_fit", "ipf_fit_device", "SCALE_FLOOR", "SCALE_CEIL"]

SCALE_FLOOR = 1e-100
SCALE_CEIL = 1e100


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
