"""GPU parity: every device stage against the reference's golden vectors and the
CPU oracle, through the C-ABI library (libgridot_b200.so).

Bars (BASELINE.json): fp64 mode -- SumPool, C-bar, interpolation, grid
c-transforms and coarse plans bit-exact, bound raw values within 1e-9
relative (most are exact); fp32 mode -- bounds within 1e-5 relative;
lower <= upper on every pair.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import case_ids, rel_close
from oracle import port as P
from test_oracle_golden import inputs_for

pytestmark = pytest.mark.gpu

G = pytest.importorskip("paper_2506_00976_b200")


def _bits(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and a.tobytes() == b.tobytes()


SMALL = case_ids("small_cases.npz")


@pytest.mark.parametrize("idx", range(len(SMALL)), ids=SMALL)
def test_stages_bit_exact_small(small_cases, idx):
    c = small_cases[idx]
    dims, k, p = c["dims"], c["kappa"], c["p"]
    mu, nu = inputs_for(c)
    grid, spec = G.GridSpec(dims), G.CoarseningSpec(k)
    gm, gn = G.GridMeasure(grid, mu), G.GridMeasure(grid, nu)
    assert _bits(G.coarsen_measure(gm, spec).mass, c["sumpool_mu"])
    assert _bits(G.coarsen_measure(gn, spec).mass, c["sumpool_nu"])
    cb = G.weighted_cost_matrix(gm, gn, spec, p)
    assert _bits(cb.values, c["cbar"]), np.max(np.abs(cb.values - c["cbar"]))
    assert np.array_equal(cb.unused, c["cbar_unused"])
    centres = G.coarsen_grid(grid, spec)
    for meth, key in (("multilinear", "f_hat"), ("nearest", "f_hat_nearest")):
        fh = G.interpolate_potential(c["f_ext"], centres, grid, meth)
        assert _bits(fh, c[key]), meth


@pytest.mark.parametrize("idx", range(len(SMALL)), ids=SMALL)
def test_four_bounds_fp64_small(small_cases, idx):
    c = small_cases[idx]
    dims, k, p = c["dims"], c["kappa"], c["p"]
    mu, nu = inputs_for(c)
    kern = None
    if "kernel" in c:
        kern = G.UpscaleKernel(k, len(dims), c["kernel"])
    for xi, mi, name in ((None, 10_000, "pu"), (0.0, 7, "pu7")):
        reps = G.quantized_bounds(mu[None], nu[None], dims, k, p, xi=xi, max_iter=mi, kernel=kern,
                                  return_exceptions=False)[0]
        pu = reps["primal_upscaling"]
        assert rel_close(pu.value, float(c[f"{name}_value"]), 1e-9), (name, pu.value)
        assert pu.iterations == int(c[f"{name}_iterations"])
        assert pu.components["converged"] == float(c[f"{name}_converged"])
        for key in ("transport", "delta_mu", "delta_nu"):
            assert rel_close(pu.components[key], float(c[f"{name}_{key}"]), 1e-9), key
    assert rel_close(reps["weighted_cost"].value, float(c["wc_value"]), 1e-12)
    assert rel_close(reps["min_cost"].raw_value, float(c["mc_raw"]), 1e-12)  # warm-started LP
    assert rel_close(reps["dual_upscaling"].raw_value, float(c["du_multilinear_raw"]), 1e-9)
    du_n = G.dual_upscaling_lower_bound(G.GridMeasure(G.GridSpec(dims), mu),
                                        G.GridMeasure(G.GridSpec(dims), nu), k, p, "nearest")
    assert rel_close(du_n.raw_value, float(c["du_nearest_raw"]), 1e-9)
    lo = max(reps["min_cost"].value, reps["dual_upscaling"].value)
    hi = min(reps["weighted_cost"].value, reps["primal_upscaling"].value)
    assert lo <= hi + 1e-12


def test_grid_ctransform_bit_exact(small_cases):
    from paper_2506_00976_b200.device import to_dev, to_host
    from paper_2506_00976_b200.engine import ctransform_pair

    for c in small_cases:
        dims, p = c["dims"], c["p"]
        f_hat = to_dev(c["f_hat"][None])
        mu, nu = inputs_for(c)
        f, g, dots = ctransform_pair(f_hat, to_dev(mu[None]), to_dev(nu[None]), dims, p, "fp64")
        assert _bits(to_host(g)[0], c["g_fine"]), c["tag"]
        assert _bits(to_host(f)[0], c["f_fine"]), c["tag"]


def test_point_ctransform_matches_oracle():
    rng = np.random.default_rng(13)
    for p in (1.0, 2.0, 1.5):
        xs, xt = rng.random((57, 2)) * 8, rng.random((41, 2)) * 8
        cost = G.CostSpec(xs, xt, p)
        f = rng.normal(size=57)
        got = G.c_transform(f, cost, "target")
        ref = P.ctransform(f, xs, xt, p, "target")
        assert np.allclose(got, ref, rtol=0, atol=1e-12) if p == 1.5 else _bits(got, ref)
        g = rng.normal(size=41)
        got = G.c_transform(g, cost, "source")
        ref = P.ctransform(g, xs, xt, p, "source")
        assert np.allclose(got, ref, rtol=0, atol=1e-12) if p == 1.5 else _bits(got, ref)
    grid = G.GridSpec((2,))
    X = grid.coordinates()
    out = G.c_transform(np.array([0.0, 5.0]), G.CostSpec(X, X, 1.0), "target")
    assert out.tolist() == [-4.0, -5.0]  # test_bounds.py:410-419


def test_fp32_mode_within_1e5(small_cases):
    for c in small_cases:
        if "kernel" in c:
            continue
        dims, k, p = c["dims"], c["kappa"], c["p"]
        mu, nu = inputs_for(c)
        reps = G.quantized_bounds(mu[None], nu[None], dims, k, p, precision="fp32",
                                  return_exceptions=False)[0]
        assert rel_close(reps["weighted_cost"].value, float(c["wc_value"]), 1e-5), c["tag"]
        assert rel_close(reps["primal_upscaling"].value, float(c["pu_value"]), 1e-5), c["tag"]
        assert rel_close(reps["dual_upscaling"].raw_value, float(c["du_multilinear_raw"]),
                         1e-5), c["tag"]
        assert rel_close(reps["min_cost"].raw_value, float(c["mc_raw"]), 1e-12)  # warm-started LP


def test_ring_fallback_kat(small_cases):
    c = next(x for x in small_cases if x["tag"] == "ring_fallback")
    mu, nu = inputs_for(c)
    grid = G.GridSpec(c["dims"])
    rep = G.primal_upscaling_upper_bound(G.GridMeasure(grid, mu), G.GridMeasure(grid, nu), 2,
                                         1.0, kernel=G.UpscaleKernel(2, 1, c["kernel"]))
    assert rep.value == pytest.approx(3.0, abs=1e-9)
    assert rep.components["converged"] == 1.0


def test_dirac_kats():
    grid = G.GridSpec((4, 4))
    a = G.GridMeasure(grid, np.eye(1, 16, 0).ravel())
    b = G.GridMeasure(grid, np.eye(1, 16, 15).ravel())
    assert G.weighted_cost_upper_bound(a, b, 2, 2.0).value == pytest.approx(math.sqrt(18))
    pu = G.primal_upscaling_upper_bound(a, b, 2, 2.0)
    assert pu.value == pytest.approx(math.sqrt(18), abs=1e-9)
    assert pu.components["delta_mu"] == pytest.approx(0.0, abs=1e-12)
    du = G.dual_upscaling_lower_bound(a, b, 2, 2.0)
    assert 0.0 <= du.value <= math.sqrt(18) + 1e-9
    rng = np.random.default_rng(16)
    m = G.normalize(G.GridMeasure(G.GridSpec((8, 8)), rng.random(64)))
    assert G.dual_upscaling_lower_bound(m, m, 2, 2.0).value == 0.0
    assert G.min_cost_lower_bound(m, m, 2, 2.0).value == 0.0


def test_non_divisible_and_oversized_kappa_match_oracle():
    rng = np.random.default_rng(21)
    for dims, k in (((5, 3), 2), ((4, 4), 8), ((7,), 3), ((6, 5, 3), 2)):
        n = int(np.prod(dims))
        mu, nu = rng.random(n), rng.random(n)
        mu, nu = mu / mu.sum(), nu / nu.sum()
        for p in (1.0, 2.0):
            reps = G.quantized_bounds(mu[None], nu[None], dims, k, p, return_exceptions=False)[0]
            ref = P.four_bounds(mu, nu, dims, k, p)
            for m in G.QUANT_METHODS:
                assert rel_close(reps[m].raw_value, ref[m]["raw_value"], 1e-9), (dims, k, p, m)


def test_batched_equals_single_and_sandwich():
    rng = np.random.default_rng(20)
    dims = (16, 16)
    mus = rng.random((6, 256))
    nus = rng.random((6, 256))
    mus /= mus.sum(1, keepdims=True)
    nus /= nus.sum(1, keepdims=True)
    for p in (1.0, 2.0):
        batch = G.quantized_bounds(mus, nus, dims, 4, p, return_exceptions=False)
        for b in range(6):
            one = G.quantized_bounds(mus[b:b + 1], nus[b:b + 1], dims, 4, p,
                                     return_exceptions=False)[0]
            for m in G.QUANT_METHODS:
                assert batch[b][m].raw_value == one[m].raw_value
            lo = max(batch[b]["min_cost"].value, batch[b]["dual_upscaling"].value)
            hi = min(batch[b]["weighted_cost"].value, batch[b]["primal_upscaling"].value)
            assert lo <= hi


def test_ipf_fit_matches_oracle():
    import scipy.sparse as sp

    rng = np.random.default_rng(33)
    dense = rng.random((7, 5)) + 0.05
    dense[rng.random((7, 5)) < 0.3] = 0.0
    mu = rng.random(7)
    mu /= mu.sum()
    nu = rng.random(5)
    nu /= nu.sum()
    mat = sp.csr_array(dense)
    st = G.ipf_fit(mat, mu, nu, xi=1e-10)
    a, b, it, gap, conv = P.ipf(mat, mu, nu, 1e-10, 10_000)[:5]
    assert st.iterations == it and st.converged == conv
    assert _bits(st.a, a) and _bits(st.b, b)
    with pytest.raises(G.ZeroDenominatorError):
        G.ipf_fit(np.array([[1.0, 1.0], [0.0, 0.0]]), np.array([0.5, 0.5]),
                  np.array([0.5, 0.5]), xi=1e-9)


def test_weighted_tv_and_errors():
    rng = np.random.default_rng(5)
    grid = G.GridSpec((8, 8))
    a = G.normalize(G.GridMeasure(grid, rng.random(64)))
    b = G.normalize(G.GridMeasure(grid, rng.random(64)))
    w = G.tv_weights(grid, 2.0)
    ref = P.weighted_tv(a.mass, b.mass, w, 2.0)
    assert rel_close(G.weighted_tv(a, b, w, 2.0), ref, 1e-13)
    with pytest.raises(G.GridMismatchError):
        G.weighted_cost_upper_bound(a, G.GridMeasure(G.GridSpec((4, 16)), a.mass), 2, 2.0)
    with pytest.raises(G.DimensionMismatchError):
        G.primal_upscaling_upper_bound(a, b, 2, 1.0, kernel=G.UpscaleKernel.uniform(4, 2))


@pytest.mark.parametrize("dims", [(32, 32), (48, 16), (16, 8, 8), (32, 16, 8)])
@pytest.mark.parametrize("p", [1.0, 1.5])
def test_pruned_grid_ctransform_exact_fp64(dims, p):
    """Tile-pruned brute force == oracle brute force, bit for bit (fp64), on
    smooth and on rough (white-noise) potentials."""
    from paper_2506_00976_b200.device import to_dev, to_host
    from paper_2506_00976_b200.engine import ctransform_pair

    rng = np.random.default_rng(sum(dims))
    n = int(np.prod(dims))
    X = P.grid_coords(dims)
    smooth = np.sin(X[:, 0] / 5.0) * 7.0 + np.cos(X[:, 1] / 3.0) * 4.0
    for v in (smooth, rng.normal(size=n) * 10.0):
        if n > 4096 and v is not smooth:
            continue
        mass = np.full(n, 1.0 / n)
        f, g, dots = ctransform_pair(to_dev(v[None]), to_dev(mass[None]), to_dev(mass[None]),
                                     dims, p, "fp64")
        ref_g = P.ctransform(v, X, X, p, "target")
        assert _bits(to_host(g)[0], ref_g)
        ref_f = P.ctransform(ref_g, X, X, p, "source")
        assert _bits(to_host(f)[0], ref_f)


@pytest.mark.parametrize("dims", [(32, 32), (16, 8, 8)])
def test_pruned_grid_ctransform_fp32_close(dims):
    from paper_2506_00976_b200.device import to_dev, to_host
    from paper_2506_00976_b200.engine import ctransform_pair

    n = int(np.prod(dims))
    X = P.grid_coords(dims)
    v = np.sin(X[:, 0] / 5.0) * 7.0 + np.cos(X[:, 1] / 3.0) * 4.0
    mass = np.full(n, 1.0 / n)
    f, g, dots = ctransform_pair(to_dev(v[None]), to_dev(mass[None]), to_dev(mass[None]), dims,
                                 1.0, "fp32")
    ref_g = P.ctransform(v, X, X, 1.0, "target")
    assert np.max(np.abs(to_host(g)[0] - ref_g)) <= 1e-5 * max(1.0, np.abs(ref_g).max())
