"""The reference's acceptance properties, on the device path.

Ports ``pkg/tests/test_acceptance.py`` criteria 2-7 (the ones about the
quantization bounds) to this package's GPU implementation, in both precision
modes where the bound path has two:

* 2 (``:135-170``): 200 random pairs -- every lower bound <= exact <= every
  upper bound (exact = the host network simplex on the full grid problem);
* 3 (``:180-229``): strong duality of the exact solves; admissibility
  f_i + g_j <= C_ij and idempotence of the DEVICE fine potentials (the grid
  c-transform kernels the dual bound uses);
* 4 (``:233-275``): upscaled couplings have unit mass, are nonnegative and
  have bounded support;
* 5 (``:279-313``): TV correction terms below the a-priori xi cap;
* 6 (``:320-345``): mean relative error <= 10% on 32x32 gaussian pairs;
* 7 (``:352-372``): dual upscaling far faster than the exact solve.
"""

from __future__ import annotations

import math
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

G = pytest.importorskip("paper_2506_00976_b200")
from paper_2506_00976_b200 import engine as E  # noqa: E402
from paper_2506_00976_b200.device import to_dev, to_host  # noqa: E402
from paper_2506_00976_b200.harness import gen_synthetic  # noqa: E402


def _random_pair(rng, dims):
    cells = int(np.prod(dims))
    mu = G.normalize(G.GridMeasure(G.GridSpec(dims), rng.random(cells)))
    nu = G.normalize(G.GridMeasure(G.GridSpec(dims), rng.random(cells)))
    return mu, nu


def _exact(mu, nu, p):
    _, _, value = G.solve_transport(G.grid_transport_problem(mu, nu, p))
    return value ** (1.0 / p)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_criterion_2_bounds_bracket_exact_on_200_random_pairs(precision):
    rng = np.random.default_rng(1002)
    cases = []
    for _ in range(200):  # the reference's draw sequence (test_acceptance.py:140-147)
        n = int(rng.choice([8, 16]))
        d = int(rng.choice([1, 2]))
        p = float(rng.choice([1.0, 2.0]))
        kappa = int(rng.choice([2, 4]))
        mult = float(rng.choice([0.05, 0.5]))
        mu, nu = _random_pair(rng, (n,) * d)
        cases.append((n, d, p, kappa, mult, mu, nu))
    violations = []
    groups = {}
    for i, c in enumerate(cases):
        groups.setdefault(c[:4], []).append(i)
    for (n, d, p, kappa), idx in groups.items():
        mus = np.stack([cases[i][5].mass for i in idx])
        nus = np.stack([cases[i][6].mass for i in idx])
        reps = G.quantized_bounds(mus, nus, (n,) * d, kappa, p, precision=precision,
                                  return_exceptions=False)
        for i, rep in zip(idx, reps):
            _, _, _, _, mult, mu, nu = cases[i]
            exact = _exact(mu, nu, p)
            coords = mu.grid.coordinates()
            cost = G.CostSpec(coords, coords, p)
            params = G.RegularizationParams(mult * float(n) ** p, max_iter=500)
            lows = [rep["min_cost"].value, rep["dual_upscaling"].value,
                    G.reg_lower_bound(mu, nu, cost, params).value]
            highs = [rep["weighted_cost"].value, rep["primal_upscaling"].value,
                     G.reg_upper_bound(mu, nu, cost, params).value]
            for v in lows:
                if v > exact + 1e-7:
                    violations.append((i, "low", v, exact))
            for v in highs:
                if v < exact - 1e-7:
                    violations.append((i, "high", v, exact))
    assert not violations, violations[:10]


def test_criterion_3_strong_duality_of_exact_solves():
    rng = np.random.default_rng(1003)
    for _ in range(40):
        d = int(rng.integers(1, 3))
        n = int(rng.integers(2, 17 if d == 1 else 9))
        mu, nu = _random_pair(rng, (n,) * d)
        p = float(rng.choice([1.0, 1.5, 2.0]))
        problem = G.grid_transport_problem(mu, nu, p)
        _, duals, value = G.solve_transport(problem)
        dual_value = float(duals.f @ problem.supply + duals.g @ problem.demand)
        assert abs(dual_value - value) <= 1e-9 * max(1.0, abs(value))
        assert duals.feasibility_slack >= -1e-9


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("dims", [(4,), (8,), (4, 4), (8, 8), (6,), (3, 3), (16, 16), (8, 8, 8)])
@pytest.mark.parametrize("p", [1.0, 2.0])
def test_criterion_3_device_potentials_admissible_and_idempotent(dims, p, precision):
    """f_hat from the coarse duals (device interpolation), then g = T f_hat and
    f = T g through the grid c-transform kernels of the dual bound; the pair
    (f, g) must be admissible and T f must give g back."""
    rng = np.random.default_rng(1003 + sum(dims) + int(p))
    mu, nu = _random_pair(rng, dims)
    spec = G.CoarseningSpec(2)
    mu_c, nu_c = G.coarsen_measure(mu, spec), G.coarsen_measure(nu, spec)
    centers = G.coarsen_grid(mu.grid, spec)
    ctil = G.center_cost_matrix(centers, centers, p)
    problem = G.build_transport_problem(mu_c.mass, nu_c.mass, ctil.values)
    _, duals, _ = G.solve_transport(problem)
    f_ext = np.min(ctil.values[:, problem.dst_index] - duals.g[None, :], axis=1)
    f_hat = G.interpolate_potential(f_ext, centers, mu.grid)
    f, g, _ = E.ctransform_pair(to_dev(f_hat[None]), to_dev(mu.mass[None]),
                                to_dev(nu.mass[None]), dims, p, precision)
    f64, g64 = to_host(f)[0].astype(np.float64), to_host(g)[0].astype(np.float64)
    coords = mu.grid.coordinates()
    C = G.CostSpec(coords, coords, p).full()
    scale = max(1.0, float(np.abs(C).max()))
    tol = 1e-9 if precision == "fp64" else 4e-7 * scale
    assert (C - f64[:, None] - g64[None, :]).min() >= -tol
    # idempotence: the target transform of f is g again
    _, g_again, _ = E.ctransform_pair(to_dev(f64[None]), to_dev(mu.mass[None]),
                                      to_dev(nu.mass[None]), dims, p, precision)
    itol = 1e-12 if precision == "fp64" else 4e-7 * scale
    assert np.max(np.abs(to_host(g_again)[0].astype(np.float64) - g64)) <= itol
    if precision == "fp64":  # and the brute-force host definition agrees
        assert np.array_equal(g64, np.min(C - f_hat[:, None], axis=0))


def test_criterion_4_upscaled_couplings_are_valid():
    rng = np.random.default_rng(1004)
    checked = 0
    for dims in [(8, 8), (4, 4), (16, 16), (8,), (6, 6)]:
        for kappa in (2, 4):
            mu, nu = _random_pair(rng, dims)
            spec = G.CoarseningSpec(kappa)
            mu_c, nu_c = G.coarsen_measure(mu, spec), G.coarsen_measure(nu, spec)
            centers = G.coarsen_grid(mu.grid, spec)
            ctil = G.center_cost_matrix(centers, centers, 2.0)
            problem = G.build_transport_problem(mu_c.mass, nu_c.mass, ctil.values)
            coupling, _, _ = G.solve_transport(problem)
            n_c = mu_c.grid.cell_count
            full = G.SparseCoupling(row=problem.src_index[coupling.row],
                                    col=problem.dst_index[coupling.col], mass=coupling.mass,
                                    shape=(n_c, n_c))
            d = mu.grid.ndim
            kernels = [G.UpscaleKernel.uniform(kappa, d),
                       G.UpscaleKernel(kappa, d, rng.random((kappa,) * (2 * d)) + 0.01)]
            padded = spec.padded_dims(mu.grid)
            for kernel in kernels:
                fine = G.upscale_coupling(full, kernel, padded)
                checked += 1
                assert abs(fine.total_mass - 1.0) <= 1e-12
                assert fine.mass.size == 0 or fine.mass.min() >= 0.0
                assert fine.row.size <= kappa ** (2 * d) * (2 * n_c - 1)
    assert checked > 0


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_criterion_4_device_fit_keeps_marginals(precision):
    """The device never materialises the fine coupling; what it certifies is
    the IPF-fitted plan's marginals: on converged runs the L1 marginal gap is
    below xi and the transport term is a nonnegative cost."""
    rng = np.random.default_rng(1014)
    for dims, kappa in [((16, 16), 2), ((16, 16), 4), ((32,), 4), ((8, 8, 8), 2)]:
        mus = np.stack([_random_pair(rng, dims)[0].mass for _ in range(4)])
        nus = np.stack([_random_pair(rng, dims)[1].mass for _ in range(4)])
        for p in (1.0, 2.0):
            reps = G.quantized_bounds(mus, nus, dims, kappa, p, precision=precision, xi=1e-10,
                                      methods=("primal_upscaling",), return_exceptions=False)
            for rep in reps:
                pu = rep["primal_upscaling"]
                assert pu.components["converged"] == 1.0
                assert pu.components["marginal_gap"] < 1e-10
                assert pu.components["transport"] >= 0.0


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_criterion_5_correction_terms_below_cap(precision):
    rng = np.random.default_rng(1005)
    checked = 0
    for _ in range(12):
        d = int(rng.choice([1, 2]))
        n = int(rng.choice([8, 16]))
        p = float(rng.choice([1.0, 2.0]))
        xi = float(rng.choice([1e-6, 1e-8]))
        mu, nu = _random_pair(rng, (n,) * d)
        cap = 2.0 ** (2.0 - 2.0 / p) * xi ** (1.0 / p) * (0.5 * math.sqrt(d) * n)
        coords = mu.grid.coordinates()
        reg = G.reg_upper_bound(mu, nu, G.CostSpec(coords, coords, p),
                                G.RegularizationParams(0.5 * float(n) ** p, xi=xi))
        if reg.components["converged"] == 1.0:
            checked += 1
            assert reg.components["delta_mu"] + reg.components["delta_nu"] < cap
        pu = G.quantized_bounds(mu.mass[None], nu.mass[None], (n,) * d, 2, p, xi=xi,
                                precision=precision, methods=("primal_upscaling",),
                                return_exceptions=False)[0]["primal_upscaling"]
        if pu.components["converged"] == 1.0:
            checked += 1
            assert pu.components["delta_mu"] + pu.components["delta_nu"] < cap
    assert checked > 0


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_criterion_6_bound_accuracy_on_gaussian_pairs(precision):
    wc_err, du_err = [], []
    mus = np.stack([gen_synthetic("gaussians", 32, 2, 100 + i).mass for i in range(10)])
    nus = np.stack([gen_synthetic("gaussians", 32, 2, 200 + i).mass for i in range(10)])
    reps = G.quantized_bounds(mus, nus, (32, 32), 2, 2.0, precision=precision,
                              methods=("weighted_cost", "dual_upscaling"),
                              return_exceptions=False)
    grid = G.GridSpec((32, 32))
    for i, rep in enumerate(reps):
        exact = _exact(G.GridMeasure(grid, mus[i]), G.GridMeasure(grid, nus[i]), 2.0)
        wc_err.append((rep["weighted_cost"].value - exact) / exact)
        du_err.append((exact - rep["dual_upscaling"].value) / exact)
    assert float(np.mean(wc_err)) <= 0.10
    assert float(np.mean(du_err)) <= 0.10
    assert min(wc_err) >= -1e-9 and min(du_err) >= -1e-9


def test_criterion_7_dual_upscaling_speedup():
    ratios = []
    for i in range(3):
        mu = gen_synthetic("gaussians", 64, 2, 300 + i)
        nu = gen_synthetic("gaussians", 64, 2, 400 + i)
        G.dual_upscaling_lower_bound(mu, nu, 4, 2.0)  # warm (first-launch costs)
        t0 = time.perf_counter()
        G.solve_transport(G.grid_transport_problem(mu, nu, 2.0))
        t_exact = time.perf_counter() - t0
        t0 = time.perf_counter()
        G.dual_upscaling_lower_bound(mu, nu, 4, 2.0)
        ratios.append((time.perf_counter() - t0) / t_exact)
    assert float(np.median(ratios)) <= 0.25
