"""Entropic bounds (reference sinkhorn.py:150-299).

CPU: the oracle restatement (oracle/port.py reg_bounds) against the fixtures
the live reference produced (tests/golden/make_entropic_golden.py), the
parameter validation and the pair checks of the public API.
GPU (``-m gpu``): reg_lower_bound / reg_upper_bound on the device against the
same fixtures and against the oracle on larger grids.

Tolerances (fp64): the dual value (hence the lower bound) and the transport
term within 1e-9 relative.  The weighted-TV corrections are 2^(1-1/p) I^(1/p)
of an inner sum I = sum_i w_i |hat_i - marg_i| that cancels to rounding noise
once the fit is tight, so they are compared through I with an absolute
tolerance of 1e-12 * sum_i w_i marg_i (the rounding of the marginals), and the
upper bound within 1e-9 of the transport term plus that tolerance carried
through the root.
"""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

import paper_2506_00976_b200 as G
from oracle import port as P

Z = np.load(os.path.join(os.path.dirname(__file__), "golden", "entropic.npz"))
META = json.loads(str(Z["meta"]))
IDS = [m["tag"] for m in META]


def _inputs(q):
    return Z[f"c{q}_mu"], Z[f"c{q}_nu"], META[q]


def _inner(delta, p):
    return (delta / 2.0 ** (1.0 - 1.0 / p)) ** p


def _close(got, want, rel=1e-9):
    return abs(got - want) <= rel * max(1.0, abs(want))


@pytest.mark.parametrize("q", range(len(META)), ids=IDS)
def test_oracle_matches_reference_fixtures(q):
    mu, nu, m = _inputs(q)
    r = P.reg_bounds(mu, nu, tuple(m["dims"]), m["p"], m["eps"], m["xi"], m["max_iter"])
    assert r["log_domain"] == m["log_domain"]
    for side in ("lower", "upper"):
        for k, v in m[side].items():
            assert _close(r[side][k], v, 1e-12), (side, k, r[side][k], v)


def test_params_validation():
    with pytest.raises(ValueError):
        G.RegularizationParams(epsilon=0.0)
    with pytest.raises(ValueError):
        G.RegularizationParams(epsilon=1.0, xi=0.0)
    with pytest.raises(ValueError):
        G.RegularizationParams(epsilon=1.0, max_iter=0)
    p = G.RegularizationParams(0.5)
    assert p.xi is None and p.max_iter == 10_000 and p.resolve_xi(10) == 1e-8


def _grid_cost(grid, p):
    X = grid.coordinates()
    return G.CostSpec(X, X, p)


def test_pair_checks_raise_before_any_device_work():
    g1, g2 = G.GridSpec((3,)), G.GridSpec((4,))
    a = G.GridMeasure(g1, np.ones(3) / 3)
    b = G.GridMeasure(g2, np.ones(4) / 4)
    params = G.RegularizationParams(1.0)
    with pytest.raises(G.GridMismatchError):
        G.reg_lower_bound(a, b, _grid_cost(g1, 2.0), params)
    with pytest.raises(G.DimensionMismatchError):
        G.reg_upper_bound(a, a, _grid_cost(g2, 2.0), params)
    big = G.GridSpec((257, 256))
    m = G.GridMeasure(big, np.ones(big.cell_count) / big.cell_count)
    X = np.zeros((big.cell_count, 2))
    with pytest.raises(G.KernelSizeError):
        G.reg_lower_bound(m, m, G.CostSpec(X, X, 2.0), params)
    c = G.GridMeasure(g1, np.array([0.5, 0.5, 0.1]))
    with pytest.raises(G.UnbalancedError):
        G.reg_lower_bound(a, c, _grid_cost(g1, 2.0), params)


def _check(rep_lo, rep_up, want, mu, nu, dims, p):
    lo, up = want["lower"], want["upper"]
    assert _close(rep_lo.components["dual_value"], lo["dual_value"])
    assert _close(rep_lo.raw_value, lo["raw_value"])
    assert rep_lo.value == max(0.0, rep_lo.raw_value)
    assert _close(rep_up.components["transport"], up["transport"])
    w = P.tv_weights(dims, p)
    slack = 1e-9 * max(1.0, abs(up["transport"]))
    for key, marg in (("delta_mu", mu), ("delta_nu", nu)):
        tol = 1e-12 * float(w @ marg)
        inner = _inner(up[key], p)
        assert abs(_inner(rep_up.components[key], p) - inner) <= tol, key
        # the same tolerance carried through the root 2^(1-1/p) I^(1/p)
        root = lambda x: 2.0 ** (1.0 - 1.0 / p) * x ** (1.0 / p)  # noqa: E731
        slack += root(inner + tol) - root(max(inner - tol, 0.0))
    assert abs(rep_up.value - up["value"]) <= slack
    assert rep_up.value == pytest.approx(sum(rep_up.components[k] for k in
                                             ("transport", "delta_mu", "delta_nu")), rel=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("q", range(len(META)), ids=IDS)
def test_device_matches_reference_fixtures(q):
    mu, nu, m = _inputs(q)
    dims, p = tuple(m["dims"]), m["p"]
    grid = G.GridSpec(dims)
    params = G.RegularizationParams(m["eps"], xi=m["xi"], max_iter=m["max_iter"])
    a, b = G.GridMeasure(grid, mu), G.GridMeasure(grid, nu)
    lo = G.reg_lower_bound(a, b, _grid_cost(grid, p), params)
    up = G.reg_upper_bound(a, b, _grid_cost(grid, p), params)
    assert lo.method == "reg_lower" and up.method == "reg_upper"
    assert lo.iterations == m["lower"]["iterations"] and up.iterations == lo.iterations
    assert lo.components["converged"] == m["lower"]["converged"]
    _check(lo, up, m, mu, nu, dims, p)


@pytest.mark.gpu
@pytest.mark.parametrize("dims,p,eps,holes", [((48, 48), 2.0, 0.02 * 48 ** 2, 0.0),
                                              ((40, 36), 1.0, 0.5, 0.2),
                                              ((12, 12, 12), 2.0, 0.1 * 144, 0.0)])
def test_device_matches_oracle_larger(dims, p, eps, holes):
    rng = np.random.default_rng(hash(dims) % 1000)
    n = int(np.prod(dims))
    mu, nu = rng.random(n), rng.random(n)
    if holes:
        mu[rng.random(n) < holes] = 0.0
        nu[rng.random(n) < holes] = 0.0
    mu, nu = mu / mu.sum(), nu / nu.sum()
    want = P.reg_bounds(mu, nu, dims, p, eps, None, 2000)
    grid = G.GridSpec(dims)
    params = G.RegularizationParams(eps, max_iter=2000)
    a, b = G.GridMeasure(grid, mu), G.GridMeasure(grid, nu)
    lo = G.reg_lower_bound(a, b, _grid_cost(grid, p), params)
    up = G.reg_upper_bound(a, b, _grid_cost(grid, p), params)
    assert abs(lo.iterations - want["lower"]["iterations"]) <= 1
    _check(lo, up, want, mu, nu, dims, p)


@pytest.mark.gpu
def test_device_full_size_brackets_quantization_bounds():
    """128 x 128 (16384 cells, a 2 GB kernel): the entropic bracket holds and
    contains the quantization bracket's certified interval's overlap."""
    from paper_2506_00976_b200 import synthetic as S

    dims = (128, 128)
    mu, nu = S.measure(3, 0, 0), S.measure(3, 0, 1)
    grid = G.GridSpec(dims)
    a, b = G.GridMeasure(grid, mu), G.GridMeasure(grid, nu)
    params = G.RegularizationParams(0.05 * 128 ** 2, max_iter=500)
    lo = G.reg_lower_bound(a, b, _grid_cost(grid, 2.0), params)
    up = G.reg_upper_bound(a, b, _grid_cost(grid, 2.0), params)
    q = G.quantized_bounds(mu[None], nu[None], dims, 4, 2.0)[0]
    qlo = max(q["min_cost"].value, q["dual_upscaling"].value)
    qhi = min(q["weighted_cost"].value, q["primal_upscaling"].value)
    assert lo.value <= up.value
    assert lo.value <= qhi * (1 + 1e-9) and qlo <= up.value * (1 + 1e-9)


@pytest.mark.gpu
def test_device_kernel_cap_size():
    """The reference's cap (2^16 cells, a 34 GB fp64 kernel) on one B200:
    256 x 256, p = 2.  No CPU oracle at this size; the bounds must bracket
    the quantization bracket's overlap."""
    from paper_2506_00976_b200 import synthetic as S

    dims = (256, 256)
    mu, nu = S.measure(4, 0, 0), S.measure(4, 0, 1)
    grid = G.GridSpec(dims)
    a, b = G.GridMeasure(grid, mu), G.GridMeasure(grid, nu)
    params = G.RegularizationParams(0.02 * 256 ** 2, max_iter=200)
    lo = G.reg_lower_bound(a, b, _grid_cost(grid, 2.0), params)
    up = G.reg_upper_bound(a, b, _grid_cost(grid, 2.0), params)
    q = G.quantized_bounds(mu[None], nu[None], dims, 8, 2.0)[0]
    qlo = max(q["min_cost"].value, q["dual_upscaling"].value)
    qhi = min(q["weighted_cost"].value, q["primal_upscaling"].value)
    assert 0.0 <= lo.value <= up.value
    assert lo.value <= qhi * (1 + 1e-9) and qlo <= up.value * (1 + 1e-9)
