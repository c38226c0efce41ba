"""Pin the CPU oracle to golden vectors produced by the live reference.

The oracle (oracle/port.py + oracle/simplex_oracle.c) is the checker for
every GPU parity test; these CPU tests prove it reproduces the reference bit
for bit on the committed fixtures (tests/golden/make_golden.py).
"""

from __future__ import annotations

import hashlib
import os

import numpy as np
import pytest

from conftest import case_ids
from oracle import port as P
from paper_2506_00976_b200 import synthetic as S

FULL = os.environ.get("GRIDOT_FULL") == "1"


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def inputs_for(case):
    if "mu" in case:
        return np.asarray(case["mu"]), np.asarray(case["nu"])
    mu, nu = S.measure(case["cfg"], case["pair"], 0), S.measure(case["cfg"], case["pair"], 1)
    assert _sha(mu) == str(case["mu_sha"]) and _sha(nu) == str(case["nu_sha"]), \
        "synthetic generator drifted from the golden fixture"
    return mu, nu


def _eq(a, b):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape and a.tobytes() == b.tobytes(), np.max(np.abs(a - b))


@pytest.mark.parametrize("idx", range(len(case_ids("small_cases.npz"))),
                         ids=case_ids("small_cases.npz"))
def test_oracle_small_case_bit_exact(small_cases, idx):
    c = small_cases[idx]
    dims, k, p = c["dims"], c["kappa"], c["p"]
    mu, nu = inputs_for(c)
    _eq(P.sumpool(mu, dims, k), c["sumpool_mu"])
    _eq(P.sumpool(nu, dims, k), c["sumpool_nu"])
    vals, unused = P.weighted_cost(mu, nu, dims, k, p)
    _eq(vals, c["cbar"])
    assert np.array_equal(unused, c["cbar_unused"])
    _eq(P.min_cost(dims, k, p), c["cmin"])
    rows, cols, mass, prob, u, v, _ = P.coarse_centre_solve(mu, nu, dims, k, p)
    _eq(rows, c["plan_row"].astype(np.int64))
    _eq(cols, c["plan_col"].astype(np.int64))
    _eq(mass, c["plan_mass"])
    _eq(u, c["plan_u"])
    _eq(v, c["plan_v"])
    assert P.weighted_cost_bound(mu, nu, dims, k, p)["value"] == float(c["wc_value"])
    assert P.min_cost_bound(mu, nu, dims, k, p)["raw_value"] == float(c["mc_raw"])
    kernel = c.get("kernel")
    for name, xi, mi in (("pu", None, 10_000), ("pu7", 0.0, 7)):
        o = P.primal_bound(mu, nu, dims, k, p, xi=xi, kernel=kernel, max_iter=mi)
        for key in ("transport", "delta_mu", "delta_nu", "marginal_gap", "converged"):
            assert o[key] == float(c[f"{name}_{key}"]), (name, key)
        assert o["iterations"] == int(c[f"{name}_iterations"])
    for meth in ("multilinear", "nearest"):
        o = P.dual_bound(mu, nu, dims, k, p, method=meth)
        assert o["raw_value"] == float(c[f"du_{meth}_raw"])
    o = P.dual_bound(mu, nu, dims, k, p)
    _eq(o["f_hat"], c["f_hat"])
    _eq(o["g"], c["g_fine"])
    _eq(o["f"], c["f_fine"])


def test_oracle_ring_fallback_kat(small_cases):
    """test_bounds.py:312-322: a zero kernel entry forces the one-ring respread."""
    c = next(x for x in small_cases if x["tag"] == "ring_fallback")
    mu, nu = inputs_for(c)
    o = P.primal_bound(mu, nu, c["dims"], c["kappa"], c["p"], kernel=c["kernel"])
    assert o["ring"]
    assert abs(o["value"] - 3.0) <= 1e-9


@pytest.mark.parametrize("tag", ["cfg1_pair0_k4_p2", "cfg2_pair0_k4_p2", "cfg3_pair0_k8_p2"]
                         + (["cfg3_pair0_k4_p1", "cfg3_pair0_k4_p2", "cfg3_pair0_k8_p1",
                             "cfg5_pair0_k4_p2"] if FULL else []))
def test_oracle_config_bounds_bit_exact(config_cases, tag):
    c = next(x for x in config_cases if x["tag"] == tag)
    mu, nu = inputs_for(c)
    dims, k, p = c["dims"], c["kappa"], c["p"]
    xi = None if float(c["xi"]) < 0 else float(c["xi"])
    out = P.four_bounds(mu, nu, dims, k, p, xi=xi, max_iter=int(c["max_iter"]), share_lp=True)
    assert out["weighted_cost"]["value"] == float(c["wc_value"])
    assert out["min_cost"]["raw_value"] == float(c["mc_raw"])
    assert out["primal_upscaling"]["value"] == float(c["pu_value"])
    assert out["primal_upscaling"]["iterations"] == int(c["pu_iterations"])
    assert out["dual_upscaling"]["raw_value"] == float(c["du_multilinear_raw"])


def test_pairwise_restatement_matches_numpy():
    rng = np.random.default_rng(3)
    for n in (1, 3, 7, 8, 9, 16, 17, 64, 100, 128, 129, 300, 1000):
        x = rng.random((5, n)) * rng.random((5, n))
        assert np.array_equal(P.np_pairwise(x), x.sum(axis=1))


def test_sumpool_restatement_matches_add_at():
    rng = np.random.default_rng(4)
    for dims, k in (((12, 8), 4), ((9, 10), 4), ((6, 4, 4), 2), ((7,), 3)):
        m = rng.random(int(np.prod(dims)))
        out = np.zeros(int(np.prod(P.coarse_dims(dims, k))))
        np.add.at(out, P.block_ids(dims, k), m)
        assert out.tobytes() == P.sumpool(m, dims, k).tobytes()


@pytest.mark.parametrize("cfg", [2, 3, 4, 5])
def test_batch_golden_pins_the_generator(cfg):
    """tests/golden/batch_cfg*.npz (reference values for every benched pair)
    were made from these exact masses: the GPU box regenerates them from seeds."""
    import json

    from conftest import GOLDEN

    z = np.load(os.path.join(GOLDEN, f"batch_cfg{cfg}.npz"), allow_pickle=False)
    meta = json.loads(str(z["meta"]))
    assert meta["pairs"] == (64 if cfg == 5 else 45)
    assert [tuple(c) for c in meta["combos"]] == [(int(k), float(p))
                                                  for k, p in S.WORKLOADS[cfg].combos]
    for b in range(0, meta["pairs"], 11):
        for side, key in ((0, "mu_sha"), (1, "nu_sha")):
            m = S.measure(cfg, b, side)
            assert hashlib.sha256(np.ascontiguousarray(m).tobytes()).hexdigest() == \
                str(z[key][b])
