"""ORACLE / TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference.

This module restates, in numpy (+ the C simplex in ``simplex_oracle.c``), the
algorithm of the reference package ``gridot`` for the four quantization bounds
(``pkg/src/gridot/quantized.py``) and the primitives they call.  It exists to
CHECK the B200 product (``paper_2506_00976_b200``): only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline leg and
``--impl reference``) may import it.  The product never imports it.

Parity is pinned: ``tests/test_oracle_golden.py`` compares every function here
against fixtures that ``tests/golden/make_golden.py`` produced by running the
live reference (``/root/reference/pkg/src``) in the build container.

Floating-point order notes (all verified against the reference, see the tests):
  * SumPool adds in ascending fine flat index per block (np.add.at order,
    measures.py:257-267).
  * C-bar: per column c, sequential sum over the block's rows of (C*mu_r)*nu_c,
    then numpy's 8-lane pairwise sum over the block's columns (costs.py:151-170).
  * IPF uses CSR products with canonical (sorted) column indices -- per-row
    sequential sums in ascending column, per-column sequential sums in
    ascending row (sinkhorn.py:120-136, quantized.py:322-333).
"""

from __future__ import annotations

import ctypes
import itertools
import math
import os
import subprocess

import numpy as np
import scipy.sparse as sp

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle_simplex.so")


class OracleError(Exception):
    """Any failure the reference would raise as a GridotError subclass."""


class ZeroDenominator(OracleError):
    pass


class Overflow(OracleError):
    pass


class PivotLimit(OracleError):
    pass


# ---------------------------------------------------------------------------
# grid helpers (measures.py:45-130, 236-281)
# ---------------------------------------------------------------------------


def cell_count(dims) -> int:
    return int(np.prod(dims))


def grid_coords(dims) -> np.ndarray:
    """1-based coordinates, flat order axis-1 fastest (measures.py:67-73)."""
    n = cell_count(dims)
    idx = np.unravel_index(np.arange(n), tuple(dims), order="F")
    return np.stack(idx, axis=1).astype(np.float64) + 1.0


def padded_dims(dims, kappa):
    return tuple(kappa * ((n + kappa - 1) // kappa) for n in dims)


def coarse_dims(dims, kappa):
    return tuple(p // kappa for p in padded_dims(dims, kappa))


def block_ids(dims, kappa) -> np.ndarray:
    """Coarse flat id of every fine cell (measures.py:248-254)."""
    cd = coarse_dims(dims, kappa)
    idx = np.unravel_index(np.arange(cell_count(dims)), tuple(dims), order="F")
    return np.ravel_multi_index(tuple(a // kappa for a in idx), cd, order="F")


def pad_mass(mass, dims, kappa):
    pd = padded_dims(dims, kappa)
    if pd == tuple(dims):
        return np.asarray(mass, dtype=np.float64), tuple(dims)
    t = np.asarray(mass, dtype=np.float64).reshape(dims, order="F")
    t = np.pad(t, [(0, q - n) for q, n in zip(pd, dims)])
    return t.ravel(order="F"), pd


def sumpool(mass, dims, kappa) -> np.ndarray:
    """Block sums, sequential in ascending fine index (measures.py:257-267).

    Restated with explicit offsets: for each block the within-block offsets
    are visited in ascending flat order (last axis slowest), adding into a
    zero-initialised accumulator -- the order np.add.at uses.
    """
    pm, pd = pad_mass(mass, dims, kappa)
    cd = coarse_dims(dims, kappa)
    d = len(dims)
    shape = []
    for n in cd:
        shape.extend([kappa, n])
    t = pm.reshape(shape, order="F")
    out = np.zeros(cd, dtype=np.float64, order="F")
    for off in itertools.product(range(kappa), repeat=d):
        o = off[::-1]  # product varies its last element fastest -> axis 0 fastest
        sel = []
        for a in range(d):
            sel.extend([o[a], slice(None)])
        out = out + t[tuple(sel)]
    return out.ravel(order="F")


def block_centres(dims, kappa) -> np.ndarray:
    """kappa*b + (kappa+1)/2 per axis, coarse flat order (measures.py:270-281)."""
    cd = coarse_dims(dims, kappa)
    idx = np.unravel_index(np.arange(cell_count(cd)), cd, order="F")
    return np.stack(idx, axis=1).astype(np.float64) * kappa + (kappa + 1) / 2.0


# ---------------------------------------------------------------------------
# costs (costs.py:44-53, 121-192)
# ---------------------------------------------------------------------------


def sq_dist(xa, xb) -> np.ndarray:
    """Sequential sum over axes of squared differences (scipy cdist order)."""
    out = np.zeros((xa.shape[0], xb.shape[0]))
    for a in range(xa.shape[1]):
        df = xa[:, a][:, None] - xb[:, a][None, :]
        out = out + df * df
    return out


def power_cost(sq, p):
    """rho**p from squared distances: p=2 as is, p=1 sqrt, else pow(p/2)."""
    if p == 2.0:
        return sq
    if p == 1.0:
        return np.sqrt(sq)
    return sq ** (p / 2.0)


def costs(xa, xb, p):
    return power_cost(sq_dist(xa, xb), p)


def np_pairwise(a: np.ndarray) -> np.ndarray:
    """numpy's float64 pairwise summation along the last axis, restated.

    n < 8: sequential from -0.0; n <= 128: eight strided accumulators,
    combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the tail added
    sequentially; larger n: split at n/2 rounded down to a multiple of 8.
    """
    n = a.shape[-1]
    if n < 8:
        res = np.full(a.shape[:-1], -0.0)
        for i in range(n):
            res = res + a[..., i]
        return res
    if n <= 128:
        r = [a[..., j].copy() for j in range(8)]
        i = 8
        stop = n - (n % 8)
        while i < stop:
            for j in range(8):
                r[j] = r[j] + a[..., i + j]
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            res = res + a[..., i]
            i += 1
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return np_pairwise(a[..., :n2]) + np_pairwise(a[..., n2:])


def centre_cost(dims, kappa, p):
    c = block_centres(dims, kappa)
    return costs(c, c, p)


def weighted_cost(mu, nu, dims, kappa, p, k_chunk=64):
    """C-bar with the reference's rounding order (costs.py:128-171).

    Returns (values, unused)."""
    mp, pd = pad_mass(mu, dims, kappa)
    npd, _ = pad_mass(nu, dims, kappa)
    X = grid_coords(pd)
    blk = block_ids(pd, kappa)
    order = np.argsort(blk, kind="stable")  # block-contiguous, ascending inside
    nc = cell_count(coarse_dims(dims, kappa))
    m = len(order) // nc  # kappa^d
    col_x = X[order]
    col_nu = npd[order]
    rows = order.reshape(nc, m)  # rows[k, t]: t-th cell of block k
    numer = np.empty((nc, nc))
    for k0 in range(0, nc, k_chunk):
        ks = np.arange(k0, min(nc, k0 + k_chunk))
        acc = None
        for t in range(m):
            r = rows[ks, t]
            term = costs(X[r], col_x, p)
            term = term * mp[r][:, None]
            term = term * col_nu[None, :]
            acc = term if acc is None else acc + term
        numer[ks] = np_pairwise(acc.reshape(len(ks), nc, m))
    mu_c = sumpool(mu, dims, kappa)
    nu_c = sumpool(nu, dims, kappa)
    denom = mu_c[:, None] * nu_c[None, :]
    unused = denom == 0.0
    vals = np.where(unused, centre_cost(dims, kappa, p), 0.0)
    np.divide(numer, denom, out=vals, where=~unused)
    return vals, unused


def min_cost(dims, kappa, p):
    """Closed-form per-axis gap max(0, kappa|k-l|-(kappa-1)) (costs.py:174-192)."""
    cd = coarse_dims(dims, kappa)
    idx = np.unravel_index(np.arange(cell_count(cd)), cd, order="F")
    pos = np.stack(idx, axis=1).astype(np.float64)
    sq = np.zeros((pos.shape[0], pos.shape[0]))
    for a in range(len(cd)):
        g = kappa * np.abs(pos[:, a][:, None] - pos[:, a][None, :]) - (kappa - 1)
        g = np.maximum(g, 0.0)
        sq = sq + g * g
    return sq ** (p / 2.0)


# ---------------------------------------------------------------------------
# exact transport (exact.py:103-189 + _simplex.py)
# ---------------------------------------------------------------------------

_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            subprocess.run(["make", "-s", "-C", _HERE], check=True)
        lib = ctypes.CDLL(_LIB_PATH)
        f = lib.oracle_transport_simplex
        P = ctypes.c_void_p
        f.argtypes = [P, P, P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                      ctypes.c_int64, ctypes.c_double, P, P, P, P, P, P]
        f.restype = ctypes.c_int
        _lib = lib
    return _lib


def simplex(C, sup, dem, tol=1e-10, max_pivots=None):
    """Run the restated network simplex; returns (status, bi, bj, bf, u, v, pivots)."""
    C = np.ascontiguousarray(C, dtype=np.float64)
    sup = np.ascontiguousarray(sup, dtype=np.float64)
    dem = np.ascontiguousarray(dem, dtype=np.float64)
    ns, nt = C.shape
    nb = ns + nt - 1
    bi = np.empty(nb, np.int64)
    bj = np.empty(nb, np.int64)
    bf = np.empty(nb, np.float64)
    u = np.empty(ns)
    v = np.empty(nt)
    piv = ctypes.c_int64(0)
    st = _load().oracle_transport_simplex(
        C.ctypes.data, sup.ctypes.data, dem.ctypes.data, ns, nt, 0,
        0 if max_pivots is None else int(max_pivots), float(tol),
        bi.ctypes.data, bj.ctypes.data, bf.ctypes.data, u.ctypes.data,
        v.ctypes.data, ctypes.byref(piv))
    return st, bi, bj, bf, u, v, int(piv.value)


def transport_problem(supply, demand, cost):
    """Support restriction + rebalancing (exact.py:103-136)."""
    supply = np.asarray(supply, dtype=np.float64)
    demand = np.asarray(demand, dtype=np.float64)
    si = np.nonzero(supply > 0.0)[0]
    di = np.nonzero(demand > 0.0)[0]
    if si.size == 0 or di.size == 0:
        raise OracleError("empty support")
    s = supply[si].copy()
    t = demand[di].copy()
    diff = float(s.sum() - t.sum())
    if diff != 0.0:
        if abs(diff) > 1e-12:
            raise OracleError("unbalanced")
        if diff > 0:
            t[int(np.argmax(t))] += diff
        else:
            s[int(np.argmax(s))] -= diff
    sub = np.ascontiguousarray(np.asarray(cost)[np.ix_(si, di)], dtype=np.float64)
    return s, t, sub, si, di


def solve(problem, tol=1e-10):
    """(rows, cols, mass) of positive basic flows, duals u/v, value (exact.py:156-189)."""
    s, t, sub, si, di = problem
    st, bi, bj, bf, u, v, piv = simplex(sub, s, t, tol=tol)
    if st == 1:
        raise PivotLimit(f"pivot cap after {piv}")
    if st != 0:
        raise OracleError(f"simplex status {st}")
    keep = bf > 0.0
    value = float(np.sum(bf * sub[bi, bj]))
    return bi[keep].copy(), bj[keep].copy(), bf[keep].copy(), u, v, value, piv


def signed_root(x, p):
    """reports.py:9-13."""
    if x < 0.0:
        return -((-x) ** (1.0 / p))
    return x ** (1.0 / p)


# ---------------------------------------------------------------------------
# upscaling + IPF (quantized.py:57-159, 288-380; sinkhorn.py:88-142)
# ---------------------------------------------------------------------------


def normalise_kernel(w):
    w = np.asarray(w, dtype=np.float64)
    return w / float(w.sum())


def uniform_kernel(kappa, d):
    return np.full((kappa,) * (2 * d), 1.0 / kappa ** (2 * d))


def paired(w, kappa, d):
    m = kappa ** d
    return w.reshape((m, m), order="F")


def block_cells(ids, cdims, fdims, kappa):
    """Fine flat ids of each listed block's cells, (len(ids), kappa^d)."""
    d = len(cdims)
    off = np.stack(np.unravel_index(np.arange(kappa ** d), (kappa,) * d, order="F"), axis=1)
    b = np.stack(np.unravel_index(np.asarray(ids), cdims, order="F"), axis=1)
    f = b[:, None, :] * kappa + off[None, :, :]
    return np.ravel_multi_index(tuple(f[..., a] for a in range(d)), fdims, order="F")


def upscale(rows, cols, mass, W, fdims, kappa):
    """Arc-major fine triples m*W[t,s], zero weights dropped (quantized.py:119-159)."""
    d = len(fdims)
    cd = tuple(n // kappa for n in fdims)
    R = block_cells(rows, cd, fdims, kappa)
    Cc = block_cells(cols, cd, fdims, kappa)
    Wp = paired(W, kappa, d)
    m = np.asarray(mass)[:, None, None] * Wp[None, :, :]
    r = np.broadcast_to(R[:, :, None], m.shape).ravel()
    c = np.broadcast_to(Cc[:, None, :], m.shape).ravel()
    m = m.ravel()
    k = m > 0.0
    return r[k], c[k], m[k]


def ring_spread(rows, cols, mass, cdims, fdims, kappa):
    """3^d-neighbourhood respread, duplicates summed (quantized.py:250-285)."""
    d = len(cdims)
    shifts = np.array(list(itertools.product((-1, 0, 1), repeat=d)))
    cdarr = np.array(cdims)

    def ring(fid):
        base = np.array(np.unravel_index(fid, cdims, order="F"))
        cand = base[None, :] + shifts
        ok = np.all((cand >= 0) & (cand < cdarr[None, :]), axis=1)
        cand = cand[ok]
        return np.ravel_multi_index(tuple(cand[:, a] for a in range(d)), cdims, order="F")

    R, C, M = [], [], []
    for cr, cc, cm in zip(rows, cols, mass):
        rc = block_cells(ring(cr), cdims, fdims, kappa).ravel()
        ccc = block_cells(ring(cc), cdims, fdims, kappa).ravel()
        share = cm / (rc.size * ccc.size)
        rr, c2 = np.meshgrid(rc, ccc, indexing="ij")
        R.append(rr.ravel())
        C.append(c2.ravel())
        M.append(np.full(rr.size, share))
    n = cell_count(fdims)
    mat = sp.coo_array((np.concatenate(M), (np.concatenate(R), np.concatenate(C))), shape=(n, n))
    mat.sum_duplicates()
    return mat.coords[0], mat.coords[1], mat.data


def _range_check(vec, label):
    pos = vec[vec > 0.0]
    if pos.size == 0:
        return
    lo = float(pos.min())
    hi = float(pos.max())
    if lo < 1e-100 or hi > 1e100 or not np.isfinite(hi):
        raise Overflow(f"{label} out of range")


def ipf(mat, mu, nu, xi, max_iter):
    """Alternating scaling on a CSR kernel (sinkhorn.py:101-142).

    Returns (a, b, iterations, gap, converged, kb, kta)."""
    mu = np.asarray(mu, dtype=np.float64)
    nu = np.asarray(nu, dtype=np.float64)
    matT = mat.T
    b = np.ones_like(nu)
    kb = mat @ b
    a = np.zeros_like(mu)
    kta = np.zeros_like(nu)
    gap = np.inf
    for it in range(1, max_iter + 1):
        if np.any((kb <= 0.0) & (mu > 0.0)):
            raise ZeroDenominator("row")
        a = np.divide(mu, kb, out=np.zeros_like(mu), where=kb > 0.0)
        kta = matT @ a
        if np.any((kta <= 0.0) & (nu > 0.0)):
            raise ZeroDenominator("col")
        b = np.divide(nu, kta, out=np.zeros_like(nu), where=kta > 0.0)
        kb = mat @ b
        _range_check(a, "a")
        _range_check(b, "b")
        gap = float(np.abs(a * kb - mu).sum() + np.abs(nu - b * kta).sum())
        if gap < xi:
            return a, b, it, gap, True, kb, kta
    return a, b, max_iter, gap, False, kb, kta


def tv_weights(dims, p):
    X = grid_coords(dims)
    c = (np.asarray(dims, dtype=np.float64) + 1.0) / 2.0
    df = X - c[None, :]
    return np.sum(df * df, axis=1) ** (p / 2.0)


def weighted_tv(a, b, w, p):
    inner = float(w @ np.abs(a - b))
    return 2.0 ** (1.0 - 1.0 / p) * inner ** (1.0 / p)


def coarse_centre_solve(mu, nu, dims, kappa, p):
    """SumPool + C-tilde + LP with full coarse ids (quantized.py:231-247)."""
    mu_c = sumpool(mu, dims, kappa)
    nu_c = sumpool(nu, dims, kappa)
    ctil = centre_cost(dims, kappa, p)
    prob = transport_problem(mu_c, nu_c, ctil)
    r, c, m, u, v, value, _ = solve(prob)
    si, di = prob[3], prob[4]
    return si[r], di[c], m, prob, u, v, ctil


# ---------------------------------------------------------------------------
# the four bounds (quantized.py:172-223, 288-380, 487-521)
# ---------------------------------------------------------------------------


def weighted_cost_bound(mu, nu, dims, kappa, p):
    mu_c = sumpool(mu, dims, kappa)
    nu_c = sumpool(nu, dims, kappa)
    cbar, _ = weighted_cost(mu, nu, dims, kappa, p)
    value = solve(transport_problem(mu_c, nu_c, cbar))[5]
    v = value ** (1.0 / p)
    return {"value": v, "raw_value": v, "transport": v}


def min_cost_bound(mu, nu, dims, kappa, p):
    mu_c = sumpool(mu, dims, kappa)
    nu_c = sumpool(nu, dims, kappa)
    value = solve(transport_problem(mu_c, nu_c, min_cost(dims, kappa, p)))[5]
    raw = signed_root(value, p)
    return {"value": max(0.0, raw), "raw_value": raw, "transport": raw}


def primal_bound(mu, nu, dims, kappa, p, xi=None, kernel=None, max_iter=10_000,
                 coarse=None):
    d = len(dims)
    W = uniform_kernel(kappa, d) if kernel is None else normalise_kernel(kernel)
    if coarse is None:
        coarse = coarse_centre_solve(mu, nu, dims, kappa, p)
    rows, cols, mass = coarse[0], coarse[1], coarse[2]
    mp, pd = pad_mass(mu, dims, kappa)
    npd, _ = pad_mass(nu, dims, kappa)
    n = cell_count(pd)
    src = np.nonzero(mp > 0.0)[0]
    dst = np.nonzero(npd > 0.0)[0]
    if xi is None:
        xi = 1e-9 * (src.size + dst.size)
    rpos = np.full(n, -1)
    rpos[src] = np.arange(src.size)
    cpos = np.full(n, -1)
    cpos[dst] = np.arange(dst.size)

    def fit(fr, fc, fm):
        keep = (rpos[fr] >= 0) & (cpos[fc] >= 0)
        mat = sp.csr_array((fm[keep], (rpos[fr[keep]], cpos[fc[keep]])),
                           shape=(src.size, dst.size))
        return ipf(mat, mp[src], npd[dst], xi, max_iter), mat, fr[keep], fc[keep], fm[keep]

    fr, fc, fm = upscale(rows, cols, mass, W, pd, kappa)
    ring = False
    try:
        st, mat, fr, fc, fm = fit(fr, fc, fm)
    except ZeroDenominator:
        ring = True
        cd = coarse_dims(dims, kappa)
        fr, fc, fm = ring_spread(rows, cols, mass, cd, pd, kappa)
        st, mat, fr, fc, fm = fit(fr, fc, fm)
    a, b, it, gap, conv = st[:5]
    X = grid_coords(pd)
    df = X[fr] - X[fc]
    arc_cost = np.sum(df * df, axis=1) ** (p / 2.0)
    fitted = a[rpos[fr]] * fm * b[cpos[fc]]
    transport = float(fitted @ arc_cost) ** (1.0 / p)
    mu_hat = np.zeros(n)
    mu_hat[src] = a * (mat @ b)
    nu_hat = np.zeros(n)
    nu_hat[dst] = b * (mat.T @ a)
    w = tv_weights(pd, p)
    dmu = weighted_tv(mu_hat, mp, w, p)
    dnu = weighted_tv(nu_hat, npd, w, p)
    value = transport + dmu + dnu
    return {"value": value, "raw_value": value, "transport": transport,
            "delta_mu": dmu, "delta_nu": dnu, "marginal_gap": gap,
            "converged": float(conv), "iterations": it, "ring": ring,
            "mu_hat": mu_hat, "nu_hat": nu_hat}


def interpolate(f, centres, dims, method="multilinear"):
    """d-linear interpolation with clamped extrapolation (quantized.py:388-447)."""
    vals = np.asarray(f, dtype=np.float64)
    d = len(dims)
    axes = [np.unique(centres[:, a]) for a in range(d)]
    cd = tuple(ax.size for ax in axes)
    T = vals.reshape(cd, order="F")
    Q = grid_coords(dims)
    if method == "nearest":
        idx = tuple(np.searchsorted((axes[a][:-1] + axes[a][1:]) / 2.0, Q[:, a])
                    for a in range(d))
        return T[idx]
    lo, hi, fr = [], [], []
    for a in range(d):
        ax = axes[a]
        q = Q[:, a]
        i0 = np.clip(np.searchsorted(ax, q, side="right") - 1, 0, max(ax.size - 2, 0))
        i1 = np.minimum(i0 + 1, ax.size - 1)
        span = ax[i1] - ax[i0]
        t = np.zeros_like(q)
        np.divide(q - ax[i0], span, out=t, where=span > 0.0)
        lo.append(i0)
        hi.append(i1)
        fr.append(np.clip(t, 0.0, 1.0))
    out = np.zeros(Q.shape[0])
    for corner in itertools.product((0, 1), repeat=d):
        w = np.ones(Q.shape[0])
        idx = []
        for a, side in enumerate(corner):
            w = w * (fr[a] if side else 1.0 - fr[a])
            idx.append(hi[a] if side else lo[a])
        out = out + w * T[tuple(idx)]
    return out


def ctransform(v, Xs, Xt, p, direction="target", block=1024):
    """Lazy brute-force c-transform (quantized.py:450-484)."""
    v = np.asarray(v, dtype=np.float64)
    if direction == "target":
        out = np.empty(Xt.shape[0])
        for lo in range(0, Xt.shape[0], block):
            hi = min(lo + block, Xt.shape[0])
            out[lo:hi] = np.min(costs(Xs, Xt[lo:hi], p) - v[:, None], axis=0)
        return out
    out = np.empty(Xs.shape[0])
    for lo in range(0, Xs.shape[0], block):
        hi = min(lo + block, Xs.shape[0])
        out[lo:hi] = np.min(costs(Xs[lo:hi], Xt, p) - v[None, :], axis=1)
    return out


def dual_bound(mu, nu, dims, kappa, p, method="multilinear", coarse=None):
    if coarse is None:
        coarse = coarse_centre_solve(mu, nu, dims, kappa, p)
    prob, v_dual, ctil = coarse[3], coarse[5], coarse[6]
    di = prob[4]
    f_ext = np.min(ctil[:, di] - v_dual[None, :], axis=1)
    f_hat = interpolate(f_ext, block_centres(dims, kappa), dims, method)
    X = grid_coords(dims)
    g = ctransform(f_hat, X, X, p, "target")
    f = ctransform(g, X, X, p, "source")
    dv = float(f @ np.asarray(mu) + g @ np.asarray(nu))
    raw = signed_root(dv, p)
    return {"value": max(0.0, raw), "raw_value": raw, "dual_value": dv,
            "f": f, "g": g, "f_hat": f_hat}


def four_bounds(mu, nu, dims, kappa, p, xi=None, max_iter=10_000, share_lp=False):
    """All four quantization bounds for one pair (cli.py:41 QUANT_METHODS).

    With share_lp=False each bound solves its own coarse LP, exactly as the
    reference does (the C-tilde LP runs twice); share_lp=True reuses it."""
    out = {"weighted_cost": weighted_cost_bound(mu, nu, dims, kappa, p),
           "min_cost": min_cost_bound(mu, nu, dims, kappa, p)}
    coarse = coarse_centre_solve(mu, nu, dims, kappa, p) if share_lp else None
    out["primal_upscaling"] = primal_bound(mu, nu, dims, kappa, p, xi=xi,
                                           max_iter=max_iter, coarse=coarse)
    out["dual_upscaling"] = dual_bound(mu, nu, dims, kappa, p, coarse=coarse)
    return out


# ---------------------------------------------------------------------------
# entropic bounds (sinkhorn.py:150-299): dense Gibbs kernel, log-domain restart
# ---------------------------------------------------------------------------


def _logsumexp(x, axis):
    """The reference calls scipy.special.logsumexp (scipy 1.18.1 here, the
    version the fixtures were made with); the oracle calls the same function
    so the log-domain iterates match it bit for bit."""
    from scipy.special import logsumexp

    return logsumexp(x, axis=axis)


def log_domain_scaling(cost, mu, nu, eps, xi, max_iter):
    """sinkhorn.py:150-178: the scaling iteration on potentials."""
    log_mu, log_nu = np.log(mu), np.log(nu)
    g = np.zeros_like(nu)
    lkb = _logsumexp((g[None, :] - cost) / eps, axis=1)
    f = np.zeros_like(mu)
    gap, conv, iters = np.inf, False, max_iter
    for it in range(1, max_iter + 1):
        f = eps * (log_mu - lkb)
        lkta = _logsumexp((f[:, None] - cost) / eps, axis=0)
        g = eps * (log_nu - lkta)
        lkb = _logsumexp((g[None, :] - cost) / eps, axis=1)
        mu_hat = np.exp(f / eps + lkb)
        nu_hat = np.exp(g / eps + lkta)
        gap = float(np.abs(mu_hat - mu).sum() + np.abs(nu - nu_hat).sum())
        if gap < xi:
            conv, iters = True, it
            break
    if not (np.all(np.isfinite(f)) and np.all(np.isfinite(g))):
        raise Overflow("log-domain potentials are not finite")
    return f, g, iters, gap, conv


def run_scaling(cost, mu, nu, eps, xi, max_iter):
    """sinkhorn.py:181-195: plain scaling on exp(-C/eps), log-domain restart on
    a zero denominator or scale overflow.  Returns (f, g, iterations, gap,
    converged, log_domain)."""
    try:
        K = np.exp(-cost / eps)
        a, b, it, gap, conv, _, _ = ipf(K, mu, nu, xi, max_iter)
        return eps * np.log(a), eps * np.log(b), it, gap, conv, False
    except (ZeroDenominator, Overflow):
        return (*log_domain_scaling(cost, mu, nu, eps, xi, max_iter), True)


def reg_bounds(mu, nu, dims, p, eps, xi=None, max_iter=10_000):
    """reg_lower_bound and reg_upper_bound (sinkhorn.py:226-299) of one grid
    pair with the grid cost rho^p; returns {"lower": {...}, "upper": {...},
    "log_domain": bool}."""
    mu = np.asarray(mu, dtype=np.float64)
    nu = np.asarray(nu, dtype=np.float64)
    X = grid_coords(dims)
    src, dst = np.flatnonzero(mu > 0.0), np.flatnonzero(nu > 0.0)
    mu_s, nu_s = mu[src], nu[dst]
    cost = costs(X[src], X[dst], p)
    if xi is None:
        xi = 1e-9 * (src.size + dst.size)
    f, g, it, gap, conv, logd = run_scaling(cost, mu_s, nu_s, eps, xi, max_iter)
    dv = float(f @ mu_s + g @ nu_s)
    raw = signed_root(dv, p)
    lower = {"value": max(0.0, raw), "raw_value": raw, "dual_value": dv, "marginal_gap": gap,
             "converged": float(conv), "iterations": it}
    plan = np.exp((f[:, None] + g[None, :] - cost) / eps)
    transport = float(np.sum(plan * cost)) ** (1.0 / p)
    n = cell_count(dims)
    mu_hat, nu_hat = np.zeros(n), np.zeros(n)
    mu_hat[src] = plan.sum(axis=1)
    nu_hat[dst] = plan.sum(axis=0)
    w = tv_weights(dims, p)
    dmu, dnu = weighted_tv(mu_hat, mu, w, p), weighted_tv(nu_hat, nu, w, p)
    value = transport + dmu + dnu
    upper = {"value": value, "raw_value": value, "transport": transport, "delta_mu": dmu,
             "delta_nu": dnu, "marginal_gap": gap, "converged": float(conv), "iterations": it}
    return {"lower": lower, "upper": upper, "log_domain": logd}
