"""fp32-mode device kernels against the exact fp64 kernels (GPU).

The fp32 mode of BASELINE.json only promises bounds within 1e-5 relative;
these tests pin the intermediate quantities tighter so a regression in one
kernel cannot hide behind the LP:
  * C-bar fast paths (diagonal FFMA2 tiles, Toeplitz tiles, block moments)
    vs the exact-order kernel: <= 4e-6 relative per entry (<= 64-term fp32
    chains) and identical `unused` masks;
  * fp32 pruned c-transform vs the fp64 one.
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

G = pytest.importorskip("paper_2506_00976_b200")
from paper_2506_00976_b200.costs import (centre_cost_cached, cost_table, max_sq_of,  # noqa: E402
                                         weighted_cost_batch)
from paper_2506_00976_b200.device import to_dev, to_host  # noqa: E402
from paper_2506_00976_b200.measures import sumpool_batch  # noqa: E402
from test_oracle_golden import inputs_for  # noqa: E402


def _pairs(dims, B, seed, holes=False):
    rng = np.random.default_rng(seed)
    n = int(np.prod(dims))
    mu, nu = rng.random((B, n)), rng.random((B, n))
    if holes:
        mu[rng.random((B, n)) < 0.2] = 0.0
        nu[rng.random((B, n)) < 0.2] = 0.0
    return mu / mu.sum(1, keepdims=True), nu / nu.sum(1, keepdims=True)


@pytest.mark.parametrize("dims,kappa", [((64, 64), 4), ((64, 64), 8), ((32, 48), 2),
                                        ((128, 128), 4), ((16, 16, 16), 4), ((24, 16, 8), 2),
                                        ((40, 24), 4)])
@pytest.mark.parametrize("p", [1.0, 2.0, 1.5])
def test_cbar_fast_matches_exact(dims, kappa, p):
    mu, nu = _pairs(dims, 3, hash((dims, kappa)) % 1000, holes=dims[0] == 40)
    m, v = to_dev(mu), to_dev(nu)
    mc, nc = sumpool_batch(m, dims, kappa), sumpool_batch(v, dims, kappa)
    ms = max_sq_of(dims)
    tab = to_dev(cost_table(ms, p)) if p != 2.0 else None
    ctil = to_dev(centre_cost_cached(tuple(dims), kappa, p))
    ex, ue = weighted_cost_batch(m, v, mc, nc, dims, kappa, p, 0, ctil, tab)
    fa, uf = weighted_cost_batch(m, v, mc, nc, dims, kappa, p, 1, ctil, tab)
    ex, fa = to_host(ex), to_host(fa)
    assert np.array_equal(to_host(ue), to_host(uf))
    rel = np.abs(fa - ex) / np.maximum(np.abs(ex), 1e-300)
    assert rel.max() <= 4e-6, rel.max()


@pytest.mark.parametrize("dims", [(128, 128), (32, 32, 32)])
def test_fp32_pruned_ctransform_tracks_fp64(dims):
    from paper_2506_00976_b200.engine import ctransform_pair

    rng = np.random.default_rng(7)
    n = int(np.prod(dims))
    X = np.column_stack(np.unravel_index(np.arange(n), dims, order="F")).astype(float)
    v = 5 * np.sin(X[:, 0] / 9.0) + 3 * np.cos(X[:, 1] / 7.0) + rng.normal(size=n) * 0.1
    mass = np.full(n, 1.0 / n)
    f64 = ctransform_pair(to_dev(v[None]), to_dev(mass[None]), to_dev(mass[None]), dims, 1.0,
                          "fp64")
    f32 = ctransform_pair(to_dev(v[None]), to_dev(mass[None]), to_dev(mass[None]), dims, 1.0,
                          "fp32")
    g64, g32 = to_host(f64[1])[0], to_host(f32[1]).astype(np.float64)[0]
    assert np.max(np.abs(g64 - g32)) <= 1e-5 * max(1.0, np.abs(g64).max())
    d64, d32 = to_host(f64[2]), to_host(f32[2])
    assert np.allclose(d64, d32, rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("noise", [0.1, 3.0])
def test_fp32_p1_ctransform_is_exact_brute_force(noise):
    """The fp32 p = 1 c-transform (lane-pruned table kernel on 2-D grids) equals
    the fp32 brute force min_i fl(fl(sqrt(d2)) - v_i) bit for bit: pruning only
    skips rows whose rounded lower bound cannot lower any best value."""
    import torch

    from paper_2506_00976_b200.engine import ctransform_pair

    dims = (128, 128)
    n = dims[0] * dims[1]
    rng = np.random.default_rng(int(noise * 10))
    X = np.column_stack(np.unravel_index(np.arange(n), dims, order="F")).astype(float)
    vs = []
    for b in range(2):
        v = 9 * np.sin(X[:, 0] / (7.0 + b)) + 5 * np.cos(X[:, 1] / 11.0) + \
            rng.normal(size=n) * noise
        vs.append(v)
    v64 = np.stack(vs)
    mass = np.full((2, n), 1.0 / n)
    f, g, _ = ctransform_pair(to_dev(v64), to_dev(mass), to_dev(mass), dims, 1.0, "fp32")
    Xd = torch.tensor(X, dtype=torch.float32, device="cuda")

    def brute(v32):
        out = torch.empty(n, dtype=torch.float32, device="cuda")
        for j0 in range(0, n, 2048):
            d = Xd[j0:j0 + 2048, None, :] - Xd[None, :, :]
            c = torch.sqrt((d * d).sum(-1))
            out[j0:j0 + 2048] = (c - v32[None, :]).min(dim=1).values
        return out

    for b in range(2):
        v32 = torch.tensor(v64[b], dtype=torch.float32, device="cuda")
        g_ref = brute(v32)
        assert torch.equal(g[b], g_ref)
        assert torch.equal(f[b], brute(g[b]))


@pytest.mark.parametrize("cfg,k,max_iter", [(2, 4, 40), (3, 8, 10), (4, 8, 12)])
def test_fast_ipf_tracks_exact_ipf(cfg, k, max_iter):
    """fp32-mode IPF (block-regrouped mat-vecs, ipf_fast_kernel) vs the exact
    scipy-order kernel: p = 2 prices in closed form in both modes, so the
    bounds differ only through the IPF summation order (fp64 both)."""
    from paper_2506_00976_b200 import synthetic as S

    wl = S.WORKLOADS[cfg]
    B = 6
    mus, nus = S.batch(cfg, 0, B)
    kw = dict(xi=0.0, max_iter=max_iter, methods=("primal_upscaling",), return_exceptions=False)
    ex = G.quantized_bounds(mus, nus, wl.dims, k, 2.0, precision="fp64", **kw)
    fa = G.quantized_bounds(mus, nus, wl.dims, k, 2.0, precision="fp32", **kw)
    for b in range(B):
        e, f = ex[b]["primal_upscaling"], fa[b]["primal_upscaling"]
        assert e.iterations == f.iterations == max_iter
        # the transport cost sees only the summation-order rounding; the TV
        # terms are 2^(1-1/p) tv^(1/p) of rounding-level marginal errors, so
        # their noise is amplified by the root (both ~1e-8 here)
        assert abs(e.components["transport"] - f.components["transport"]) <= \
            1e-12 * e.components["transport"]
        for key in ("delta_mu", "delta_nu"):
            assert abs(e.components[key] - f.components[key]) <= 1e-6 * max(1.0, e.value)
        assert abs(e.value - f.value) <= 1e-6 * abs(e.value), (b, e.value, f.value)


def test_fast_ipf_default_xi_and_statuses(small_cases):
    """Default xi: both IPF kernels stop on the same sweep; zero-denominator
    pairs fail the same way (ring fallback)."""
    for c in small_cases:
        if "kernel" in c:
            continue
        mu, nu = inputs_for(c)
        dims, k, p = c["dims"], c["kappa"], c["p"]
        kw = dict(methods=("primal_upscaling",), return_exceptions=True)
        e = G.quantized_bounds(mu[None], nu[None], dims, k, p, precision="fp64", **kw)[0]
        f = G.quantized_bounds(mu[None], nu[None], dims, k, p, precision="fp32", **kw)[0]
        e, f = e["primal_upscaling"], f["primal_upscaling"]
        assert type(e) is type(f), c["tag"]
        if not isinstance(e, Exception):
            assert e.iterations == f.iterations, c["tag"]
            assert abs(e.value - f.value) <= 1e-6 * abs(e.value), c["tag"]


def _f32_brute_ct(v32, dims, p):
    """fp32 emulation of the table-driven p=1 / brute-force c-transform:
    min_i (RN32(cost_ij) - v_i) with correctly rounded fp32 costs."""
    from oracle import port as P

    X = P.grid_coords(dims)
    sq = ((X[:, None, :] - X[None, :, :]) ** 2).sum(-1).astype(np.float32)
    cost = np.sqrt(sq) if p == 1.0 else sq
    return np.min(cost - v32[:, None], axis=0)


@pytest.mark.parametrize("dims", [(32, 32), (64, 48), (48, 128), (128, 16)])
def test_fp32_p1_table_ctransform_bit_exact_emulation(dims):
    """The shared-memory-table p=1 kernel computes exactly the fp32 brute
    force with correctly rounded costs (numpy float32 emulation), on smooth
    and rough potentials; the second transform too."""
    from oracle import port as P
    from paper_2506_00976_b200.engine import ctransform_pair

    rng = np.random.default_rng(dims[0] * 7 + dims[1])
    n = int(np.prod(dims))
    X = P.grid_coords(dims)
    smooth = np.sin(X[:, 0] / 5.0) * 7.0 + np.cos(X[:, 1] / 3.0) * 4.0
    for v in (smooth, rng.normal(size=n) * 10.0):
        mass = np.full(n, 1.0 / n)
        f, g, _ = ctransform_pair(to_dev(v[None]), to_dev(mass[None]), to_dev(mass[None]), dims,
                                  1.0, "fp32")
        g32 = to_host(g)[0]
        ref_g = _f32_brute_ct(v.astype(np.float32), dims, 1.0)
        assert np.array_equal(g32, ref_g)
        ref_f = _f32_brute_ct(ref_g, dims, 1.0)
        assert np.array_equal(to_host(f)[0], ref_f)


def _f32_separable_ct(v32, dims, negate_first=True):
    """fp32 emulation of the separable p=2 passes: along each axis (axis 0 =
    fastest, first pass negates), cand = RN32(d^2) + line_i, exact min."""
    a = v32.reshape(tuple(reversed(dims)))  # C-order view: last index = axis 0
    nd = len(dims)
    for ax in range(nd):
        arr_ax = nd - 1 - ax
        a = np.moveaxis(a, arr_ax, -1)
        L = a.shape[-1]
        d2 = ((np.arange(L)[:, None] - np.arange(L)[None, :]) ** 2).astype(np.float32)
        line = -a if (ax == 0 and negate_first) else a
        a = np.min(line[..., :, None] + d2, axis=-2)
        a = np.moveaxis(a.astype(np.float32), -1, arr_ax)
    return a.reshape(-1)


@pytest.mark.parametrize("dims", [(128, 128), (64, 32), (20, 12), (16, 8, 24)])
def test_fp32_separable_ctransform_bit_exact_emulation(dims):
    """Register-tiled (and, for lengths not divisible by 8, the plain) p=2
    passes equal the fp32 separable emulation bit for bit."""
    from paper_2506_00976_b200.engine import ctransform_pair

    rng = np.random.default_rng(len(dims) + dims[0])
    n = int(np.prod(dims))
    v = rng.normal(size=n) * 50.0
    mass = np.full(n, 1.0 / n)
    f, g, _ = ctransform_pair(to_dev(v[None]), to_dev(mass[None]), to_dev(mass[None]), dims, 2.0,
                              "fp32")
    ref_g = _f32_separable_ct(v.astype(np.float32), dims)
    assert np.array_equal(to_host(g)[0], ref_g)


def _all_methods(mus, nus, dims, k, p, precision, **kw):
    return G.quantized_bounds(mus, nus, dims, k, p, precision=precision, **kw)


def test_coarse_primal_matches_exact_small_cases(small_cases):
    """fp32 mode with the weighted-cost bound requested runs the coarse-level
    primal stage (primal_coarse_kernel, priced by C-bar); against the exact
    scipy-order path: same status / exception type, same sweep count, bound
    within the fp32-mode contract -- on the reference's own small inputs,
    including partial supports (zero-denominator -> ring fallback), padded
    grids, 1-D and 3-D."""
    for c in small_cases:
        if "kernel" in c:
            continue
        mu, nu = inputs_for(c)
        dims, k, p = c["dims"], c["kappa"], c["p"]
        e = _all_methods(mu[None], nu[None], dims, k, p, "fp64")[0]["primal_upscaling"]
        f = _all_methods(mu[None], nu[None], dims, k, p, "fp32")[0]["primal_upscaling"]
        assert type(e) is type(f), c["tag"]
        if not isinstance(e, Exception):
            assert e.iterations == f.iterations, c["tag"]
            assert e.components["converged"] == f.components["converged"], c["tag"]
            assert abs(e.value - f.value) <= 1e-5 * abs(e.value), (c["tag"], e.value, f.value)


@pytest.mark.parametrize("cfg,k,p,max_iter", [(2, 4, 2.0, 40), (3, 4, 1.0, 7), (3, 8, 1.0, 7),
                                              (3, 8, 2.0, 30), (4, 8, 2.0, 25),
                                              (5, 4, 2.0, 9)])
def test_coarse_primal_fixed_sweeps_tracks_exact(cfg, k, p, max_iter):
    """Fixed sweep counts (xi = 0): the coarse recursion runs every sweep;
    transport within 1e-5 (p != 2: C-bar's fp32 rounding) / 1e-12 (p = 2:
    C-bar from fp64 moments), TV terms at rounding level."""
    from paper_2506_00976_b200 import synthetic as S

    wl = S.WORKLOADS[cfg]
    B = 5
    mus, nus = S.batch(cfg, 0, B)
    kw = dict(xi=0.0, max_iter=max_iter, return_exceptions=False)
    ex = _all_methods(mus, nus, wl.dims, k, p, "fp64", **kw)
    fa = _all_methods(mus, nus, wl.dims, k, p, "fp32", **kw)
    ttol = 1e-12 if p == 2.0 else 1e-5
    for b in range(B):
        e, f = ex[b]["primal_upscaling"], fa[b]["primal_upscaling"]
        assert e.iterations == f.iterations == max_iter
        assert abs(e.components["transport"] - f.components["transport"]) <= \
            ttol * e.components["transport"], (b, e.components, f.components)
        for key in ("delta_mu", "delta_nu"):
            assert abs(e.components[key] - f.components[key]) <= 1e-6 * max(1.0, e.value)
        assert abs(e.value - f.value) <= 1e-5 * abs(e.value), (b, e.value, f.value)


def test_dadd_chain_probe_reports_a_latency():
    """gdt_probe_dadd_chain (the latency denominator of the exact IPF's unit
    sums): cycles per dependent fp64 add of one warp, a few cycles at least
    and far below a memory round trip."""
    torch = pytest.importorskip("torch")
    from paper_2506_00976_b200 import _native as N

    out = torch.zeros(1, dtype=torch.int64, device="cuda")
    for _ in range(2):
        N.check(N.lib().gdt_probe_dadd_chain(4096, N.ptr(out), None), "probe")
        torch.cuda.synchronize()
    per_add = int(out[0]) / 4096.0
    assert 2.0 < per_add < 64.0, per_add
    with pytest.raises(Exception):
        N.check(N.lib().gdt_probe_dadd_chain(4, N.ptr(out), None), "probe")


@pytest.mark.parametrize("dims,kf,kc,p", [((64, 64), 4, 8, 1.0), ((32, 32), 2, 8, 1.5),
                                           ((16, 16, 16), 2, 4, 1.0)])
def test_cbar_pooled_from_finer_level(dims, kf, kc, p):
    """gdt_weighted_cost_pool: C-bar at kappa_c from the C-bar at kappa_f (the
    numerator is additive over nested blocks).  From the exact fp64 C-bar it
    reproduces the exact C-bar at kappa_c to rounding; from the fp32-mode C-bar
    it stays inside the fp32 contract; empty blocks take the centre cost."""
    import paper_2506_00976_b200.engine as E

    rng = np.random.default_rng(7)
    N_ = int(np.prod(dims))
    mus, nus = rng.random((3, N_)), rng.random((3, N_))
    mus[0, : N_ // 3] = 0.0  # a pair with empty blocks on the source side
    nus[0, -(N_ // 4):] = 0.0
    mus /= mus.sum(1, keepdims=True)
    nus /= nus.sum(1, keepdims=True)
    for precision, tol in (("fp64", 1e-12), ("fp32", 1e-5)):
        fine = E.make_batch(mus, nus, dims, kf, p, precision=precision)
        coarse = E.make_batch(mus, nus, dims, kc, p, precision=precision)
        E._cbar(fine)
        direct = to_host(E._cbar(E.make_batch(mus, nus, dims, kc, p, precision="fp64"))[0])
        pooled = to_host(E._cbar(coarse, fine)[0])
        assert np.all(np.isfinite(pooled))
        err = np.abs(pooled - direct) / np.maximum(np.abs(direct), 1e-300)
        assert err.max() <= tol, (precision, err.max())
    # the engine picks the parent only in fp32 mode, for p != 2
    f32 = E.make_batch(mus, nus, dims, kf, p, precision="fp32")
    c32 = E.make_batch(mus, nus, dims, kc, p, precision="fp32")
    assert E.cbar_parent(c32, [f32]) is None  # not computed yet
    E._cbar(f32)
    assert E.cbar_parent(c32, [f32]) is f32
    assert E.cbar_parent(E.make_batch(mus, nus, dims, kc, p, precision="fp64"), [f32]) is None
    assert E.cbar_parent(E.make_batch(mus, nus, dims, kc, 2.0, precision="fp32"), [f32]) is None
