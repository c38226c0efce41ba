"""GPU parity at the five BASELINE.json configurations.

Golden values come from the live reference on pairs of each config
(tests/golden/configs.npz); full batches are checked through size-independent
properties (certified bracket lower <= upper on every pair, batch/single
determinism, fp32 vs fp64 agreement).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import case_ids, rel_close
from test_oracle_golden import inputs_for

pytestmark = pytest.mark.gpu

G = pytest.importorskip("paper_2506_00976_b200")
from paper_2506_00976_b200 import synthetic as S  # noqa: E402

CFG = case_ids("configs.npz")


@pytest.mark.parametrize("tag", CFG)
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_config_bounds_vs_reference(config_cases, tag, precision):
    c = next(x for x in config_cases if x["tag"] == tag)
    mu, nu = inputs_for(c)
    dims, k, p = c["dims"], c["kappa"], c["p"]
    xi = None if float(c["xi"]) < 0 else float(c["xi"])
    reps = G.quantized_bounds(mu[None], nu[None], dims, k, p, xi=xi,
                              max_iter=int(c["max_iter"]), precision=precision,
                              return_exceptions=False)[0]
    tol = 1e-9 if precision == "fp64" else 1e-5
    assert rel_close(reps["weighted_cost"].value, float(c["wc_value"]), tol)
    assert rel_close(reps["min_cost"].raw_value, float(c["mc_raw"]), 1e-12)  # warm-started LP
    assert rel_close(reps["primal_upscaling"].value, float(c["pu_value"]), tol)
    assert reps["primal_upscaling"].iterations == int(c["pu_iterations"])
    assert rel_close(reps["dual_upscaling"].raw_value, float(c["du_multilinear_raw"]), tol)
    if precision == "fp64":
        # exact C-bar; the LP is warm-started, so the optimum agrees to rounding
        assert rel_close(reps["weighted_cost"].value, float(c["wc_value"]), 1e-12)


@pytest.mark.parametrize("cfg", [2, 3, 5])
def test_full_batch_bracket_and_determinism(cfg):
    wl = S.WORKLOADS[cfg]
    B = min(wl.pairs, 16)
    mus, nus = S.batch(cfg, 0, B)
    for k, p in wl.combos[:2]:
        out = G.quantized_bounds(mus, nus, wl.dims, k, p, xi=wl.xi, max_iter=wl.max_iter,
                                 precision=wl.precision, return_exceptions=False)
        again = G.quantized_bounds(mus, nus, wl.dims, k, p, xi=wl.xi, max_iter=wl.max_iter,
                                   precision=wl.precision, return_exceptions=False)
        for b in range(B):
            lo = max(out[b]["min_cost"].value, out[b]["dual_upscaling"].value)
            hi = min(out[b]["weighted_cost"].value, out[b]["primal_upscaling"].value)
            assert lo <= hi, (cfg, k, p, b)
            for m in G.QUANT_METHODS:
                assert out[b][m].raw_value == again[b][m].raw_value


def test_fp32_tracks_fp64_on_cfg3_batch():
    wl = S.WORKLOADS[3]
    mus, nus = S.batch(3, 0, 8)
    for k, p in wl.combos:
        a = G.quantized_bounds(mus, nus, wl.dims, k, p, precision="fp64",
                               return_exceptions=False)
        b = G.quantized_bounds(mus, nus, wl.dims, k, p, precision="fp32",
                               return_exceptions=False)
        for i in range(8):
            for m in G.QUANT_METHODS:
                assert rel_close(a[i][m].raw_value, b[i][m].raw_value, 1e-5), (k, p, m)


def test_many_combos_equal_single_calls():
    """quantized_bounds_many (one LP batch for all combinations) returns the
    same values as one quantized_bounds call per combination."""
    wl = S.WORKLOADS[3]
    mus, nus = S.batch(3, 0, 6)
    many = G.quantized_bounds_many(mus, nus, wl.dims, wl.combos, precision="fp32",
                                   return_exceptions=False)
    for k, p in wl.combos:
        one = G.quantized_bounds(mus, nus, wl.dims, k, p, precision="fp32",
                                 return_exceptions=False)
        # (8, p != 2): the many-call pools C-bar from the kappa = 4 C-bar of
        # the same call (nested blocks; gdt_weighted_cost_pool), the single
        # call runs the fp32 kernel on the fine cells: both inside the fp32
        # contract, not bit-equal.  C-bar prices the weighted-cost bound and
        # the fp32-mode primal transport term.
        pooled = k == 8 and p != 2.0
        for b in range(6):
            for m in G.QUANT_METHODS:
                a_, b_ = many[(k, p)][b][m].raw_value, one[b][m].raw_value
                if pooled and m in ("weighted_cost", "primal_upscaling"):
                    assert rel_close(a_, b_, 4e-6), (k, p, b, m, a_, b_)
                else:
                    assert a_ == b_, (k, p, b, m)


@pytest.mark.parametrize("cfg,pairs", [(2, 4), (3, 3), (4, 2), (5, 4)])
def test_exact_ipf_cluster_size_invariance(cfg, pairs, monkeypatch):
    """The exact-order fp64 IPF spreads a pair over a thread-block cluster
    (ipf_cluster_kernel); every unit is still summed by one thread in the
    reference's order, so the primal bound, its components and the iteration
    count do not depend on the cluster size (1 = the single-CTA ipf_kernel)."""
    wl = S.WORKLOADS[cfg]
    mus, nus = S.batch(cfg, 0, pairs)
    k, p = wl.combos[0]
    max_iter = min(wl.max_iter, 40)
    ref = None
    for csz in (1, 2, 3, 4, 8):
        monkeypatch.setenv("GRIDOT_IPF_CLUSTER", str(csz))
        out = G.quantized_bounds(mus, nus, wl.dims, k, p, xi=0.0, max_iter=max_iter,
                                 precision="fp64", methods=("primal_upscaling",),
                                 return_exceptions=False)
        rec = [(r["primal_upscaling"].raw_value, r["primal_upscaling"].iterations,
                tuple(sorted((a, b) for a, b in r["primal_upscaling"].components.items()
                             if a != "marginal_gap")))
               for r in out]
        gaps = [r["primal_upscaling"].components.get("marginal_gap") for r in out]
        if ref is None:
            ref, ref_gaps = rec, gaps
        else:
            assert rec == ref, (cfg, csz)
            for g0, g1 in zip(ref_gaps, gaps):  # the gap folds per-CTA partials: rounding only
                if g0 is not None:
                    assert rel_close(g0, g1, 1e-12)


def test_exact_ipf_cluster_sparse_supports(monkeypatch):
    """Cluster and single-CTA exact IPF agree on measures with large empty
    regions (coarse blocks without mass, units without arcs) and on failures:
    same values or the same exception type for every pair."""
    rng = np.random.default_rng(20260)
    dims, kappa, B = (64, 64), 4, 6
    N = dims[0] * dims[1]
    mus, nus = np.zeros((B, N)), np.zeros((B, N))
    for b in range(B):
        for arr, shift in ((mus, 0), (nus, 17)):
            img = np.zeros(dims)
            # a few rectangular patches of mass; everything else exactly zero
            for _ in range(3 + b % 3):
                x0, y0 = rng.integers(0, 48, 2)
                w, h = rng.integers(3, 16, 2)
                img[x0:x0 + w, y0:y0 + h] += rng.random((min(w, 64 - x0), min(h, 64 - y0)))
            img = np.roll(img, shift, axis=b % 2)
            arr[b] = (img / img.sum()).reshape(-1, order="F")
    outs = {}
    for csz in (1, 2, 4):
        monkeypatch.setenv("GRIDOT_IPF_CLUSTER", str(csz))
        outs[csz] = G.quantized_bounds(mus, nus, dims, kappa, 2.0, xi=0.0, max_iter=30,
                                       precision="fp64", methods=("primal_upscaling",),
                                       return_exceptions=True)
    for csz in (2, 4):
        for b in range(B):
            r0, r1 = outs[1][b]["primal_upscaling"], outs[csz][b]["primal_upscaling"]
            if isinstance(r0, Exception):
                assert type(r1) is type(r0), (csz, b, r0, r1)
            else:
                assert not isinstance(r1, Exception), (csz, b, r1)
                assert r1.raw_value == r0.raw_value and r1.iterations == r0.iterations, (csz, b)



@pytest.mark.parametrize("dims,kappa,p", [((48, 40), 2, 2.0), ((24, 24, 24), 2, 1.0),
                                          ((96, 96), 8, 1.0), ((50, 46), 4, 2.0),
                                          ((64, 32), 2, 1.5)])
def test_exact_ipf_cluster_random_grids(dims, kappa, p, monkeypatch):
    """Cluster sizes 1 (single-CTA kernel), 2 and 5 on grids outside the
    benchmark shapes: kappa = 2 and 8, three dimensions, rectangular and
    non-divisible (zero-padded) grids, default xi (early convergence) -- the
    primal bound, its components and the sweep count must not depend on the
    cluster size."""
    rng = np.random.default_rng(sum(dims) * 7 + kappa)
    N_ = int(np.prod(dims))
    mus = rng.random((3, N_)) ** 3 + 1e-9
    nus = rng.random((3, N_)) ** 3 + 1e-9
    mus /= mus.sum(1, keepdims=True)
    nus /= nus.sum(1, keepdims=True)
    ref = None
    for csz in (1, 2, 5):
        monkeypatch.setenv("GRIDOT_IPF_CLUSTER", str(csz))
        out = G.quantized_bounds(mus, nus, dims, kappa, p, max_iter=60, precision="fp64",
                                 methods=("primal_upscaling",), return_exceptions=False)
        rec = [(r["primal_upscaling"].raw_value, r["primal_upscaling"].iterations,
                r["primal_upscaling"].components["transport"],
                r["primal_upscaling"].components["delta_mu"],
                r["primal_upscaling"].components["delta_nu"],
                r["primal_upscaling"].components["converged"]) for r in out]
        if ref is None:
            ref = rec
        else:
            assert rec == ref, (dims, kappa, p, csz)
