"""Generate golden fixtures by running the LIVE reference (build container only).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Writes ``tests/golden/small_cases.npz`` (inputs + reference outputs of every
hot-path function on small grids, including the reference's own known-answer
inputs) and ``tests/golden/configs.npz`` (reference bound values and coarse
C-tilde plans on pairs of the five BASELINE configs; inputs are regenerated
from seeds by ``paper_2506_00976_b200.synthetic`` and pinned by SHA-256).

``/root/reference`` does not exist on the GPU box: only this script reads it,
the committed .npz files travel instead.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.environ.get("GRIDOT_REF", "/root/reference/pkg/src"))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import gridot as G  # noqa: E402
from gridot.quantized import _solve_coarse_center  # noqa: E402

from paper_2506_00976_b200 import synthetic as S  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def coarse_plan(gm, gn, kappa, p):
    full, problem, duals, _, _, _ = _solve_coarse_center(gm, gn, G.CoarseningSpec(kappa), p)
    return full.row, full.col, full.mass, duals.f, duals.g, problem.src_index, problem.dst_index


def record_case(store, tag, dims, kappa, p, mu, nu, kernel=None, full=True, xi=None,
                max_iter=10_000):
    grid = G.GridSpec(dims)
    gm, gn = G.GridMeasure(grid, mu), G.GridMeasure(grid, nu)
    spec = G.CoarseningSpec(kappa)
    put = lambda k, v: store.__setitem__(f"{tag}/{k}", np.asarray(v))  # noqa: E731
    put("dims", np.array(dims))
    put("kappa", kappa)
    put("p", p)
    if full:
        put("mu", mu)
        put("nu", nu)
    else:
        put("mu_sha", sha(mu))
        put("nu_sha", sha(nu))
    if kernel is not None:
        put("kernel", kernel)
    if full:
        put("sumpool_mu", G.coarsen_measure(gm, spec).mass)
        put("sumpool_nu", G.coarsen_measure(gn, spec).mass)
        cb = G.weighted_cost_matrix(gm, gn, spec, p)
        put("cbar", cb.values)
        put("cbar_unused", cb.unused)
        put("cmin", G.min_cost_matrix(grid, spec, p).values)
    r, c, m, uf, ug, si, di = coarse_plan(gm, gn, kappa, p)
    put("plan_row", r)
    put("plan_col", c)
    put("plan_mass", m)
    put("plan_u", uf)
    put("plan_v", ug)
    put("plan_src", si)
    put("plan_dst", di)
    wc = G.weighted_cost_upper_bound(gm, gn, kappa, p)
    put("wc_value", wc.value)
    mc = G.min_cost_lower_bound(gm, gn, kappa, p)
    put("mc_raw", mc.raw_value)
    kern = None if kernel is None else G.UpscaleKernel(kappa, len(dims), kernel)
    runs = [("pu", xi, max_iter)] + ([("pu7", 0.0, 7)] if full else [])
    for name, xi, mi in runs:
        pu = G.primal_upscaling_upper_bound(gm, gn, kappa, p, xi=xi, kernel=kern, max_iter=mi)
        for key in ("transport", "delta_mu", "delta_nu", "marginal_gap", "converged"):
            put(f"{name}_{key}", pu.components[key])
        put(f"{name}_iterations", pu.iterations)
        put(f"{name}_value", pu.value)
    for meth in ("multilinear", "nearest") if full else ("multilinear",):
        du = G.dual_upscaling_lower_bound(gm, gn, kappa, p, method=meth)
        put(f"du_{meth}_raw", du.raw_value)
        put(f"du_{meth}_dual_value", du.components["dual_value"])
    if full:
        # dual pipeline intermediates (quantized.py:501-512)
        centres = G.coarsen_grid(grid, spec)
        ctil = G.center_cost_matrix(centres, centres, p).values
        f_ext = np.min(ctil[:, di] - ug[None, :], axis=1)
        f_hat = G.interpolate_potential(f_ext, centres, grid)
        coords = grid.coordinates()
        cost = G.CostSpec(coords, coords, p)
        g = G.c_transform(f_hat, cost, "target")
        f = G.c_transform(g, cost, "source")
        put("f_ext", f_ext)
        put("f_hat", f_hat)
        put("f_hat_nearest", G.interpolate_potential(f_ext, centres, grid, "nearest"))
        put("g_fine", g)
        put("f_fine", f)


def small_cases():
    store = {}
    index = []
    rng = np.random.default_rng(20250600)
    shapes = [((8,), 2, 1.0), ((16,), 4, 2.0), ((7,), 2, 1.0), ((8, 8), 2, 2.0),
              ((8, 8), 4, 1.0), ((6, 6), 3, 2.0), ((5, 3), 2, 2.0), ((4, 4, 4), 2, 2.0),
              ((12, 12), 4, 1.5), ((4, 4), 8, 2.0), ((16, 16), 4, 2.0), ((16, 16), 8, 1.0),
              ((6, 4, 4), 2, 1.0), ((9, 10), 4, 2.0)]
    i = 0
    for dims, kappa, p in shapes:
        for variant in ("dense", "holes"):
            n = int(np.prod(dims))
            mu, nu = rng.random(n), rng.random(n)
            if variant == "holes":
                mu[rng.random(n) < 0.3] = 0.0
                nu[rng.random(n) < 0.3] = 0.0
            mu, nu = mu / mu.sum(), nu / nu.sum()
            tag = f"s{i:02d}"
            record_case(store, tag, dims, kappa, p, mu, nu)
            index.append({"tag": tag, "dims": list(dims), "kappa": kappa, "p": p, "variant": variant})
            i += 1
    # reference known-answer inputs (pkg/tests/test_bounds.py)
    dirac = lambda n, j: np.eye(1, n, j).ravel()  # noqa: E731
    kat = [
        ("dirac_4x4", (4, 4), 2, 2.0, dirac(16, 0), dirac(16, 15), None),          # test_bounds.py:176,265
        ("dirac_line_p1", (4,), 2, 1.0, dirac(4, 0), dirac(4, 3), None),
        ("ring_fallback", (4,), 2, 1.0, dirac(4, 0), dirac(4, 3),
         np.array([[1.0, 0.0], [1.0, 1.0]])),                                        # test_bounds.py:312-322
    ]
    rk = np.random.default_rng(77)
    kat.append(("nonuniform_kernel", (8, 8), 2, 2.0, None, None, rk.random((2, 2, 2, 2)) + 0.05))
    kat.append(("nonuniform_kernel_1d", (12,), 3, 1.0, None, None, rk.random((3, 3)) + 0.01))
    for name, dims, kappa, p, mu, nu, kernel in kat:
        n = int(np.prod(dims))
        if mu is None:
            mu, nu = rk.random(n), rk.random(n)
            mu, nu = mu / mu.sum(), nu / nu.sum()
        record_case(store, name, dims, kappa, p, mu, nu, kernel=kernel)
        index.append({"tag": name, "dims": list(dims), "kappa": kappa, "p": p, "variant": "kat"})
    store["index"] = np.array(json.dumps(index))
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **store)
    print(f"small_cases: {len(index)} cases")


def config_cases():
    store = {}
    index = []
    plan = [(1, [0], True), (2, [0, 1, 2], False), (3, [0], False), (5, [0], False), (4, [0], False)]
    for cfg, pairs, full in plan:
        wl = S.WORKLOADS[cfg]
        for pi in pairs:
            mu, nu = S.measure(cfg, pi, 0), S.measure(cfg, pi, 1)
            for kappa, p in wl.combos:
                tag = f"cfg{cfg}_pair{pi}_k{kappa}_p{int(p)}"
                t0 = time.time()
                grid = G.GridSpec(wl.dims)
                gm, gn = G.GridMeasure(grid, mu), G.GridMeasure(grid, nu)
                put = lambda k, v: store.__setitem__(f"{tag}/{k}", np.asarray(v))  # noqa: E731
                if full:
                    record_case(store, tag, wl.dims, kappa, p, mu, nu, full=True, xi=wl.xi,
                                max_iter=wl.max_iter)
                else:
                    put("dims", np.array(wl.dims))
                    put("kappa", kappa)
                    put("p", p)
                    put("mu_sha", sha(mu))
                    put("nu_sha", sha(nu))
                    r, c, m, uf, ug, si, di = coarse_plan(gm, gn, kappa, p)
                    for k, v in (("plan_row", r), ("plan_col", c), ("plan_mass", m),
                                 ("plan_v", ug), ("plan_dst", di)):
                        put(k, v)
                    put("sumpool_mu", G.coarsen_measure(gm, G.CoarseningSpec(kappa)).mass)
                    put("sumpool_nu", G.coarsen_measure(gn, G.CoarseningSpec(kappa)).mass)
                    put("wc_value", G.weighted_cost_upper_bound(gm, gn, kappa, p).value)
                    put("mc_raw", G.min_cost_lower_bound(gm, gn, kappa, p).raw_value)
                    pu = G.primal_upscaling_upper_bound(gm, gn, kappa, p, xi=wl.xi, max_iter=wl.max_iter)
                    for key in ("transport", "delta_mu", "delta_nu", "marginal_gap", "converged"):
                        put(f"pu_{key}", pu.components[key])
                    put("pu_iterations", pu.iterations)
                    put("pu_value", pu.value)
                    du = G.dual_upscaling_lower_bound(gm, gn, kappa, p)
                    put("du_multilinear_raw", du.raw_value)
                    put("du_multilinear_dual_value", du.components["dual_value"])
                put("xi", -1.0 if wl.xi is None else wl.xi)
                put("max_iter", wl.max_iter)
                index.append({"tag": tag, "cfg": cfg, "pair": pi, "kappa": kappa, "p": p, "full": full})
                print(f"{tag}: {time.time() - t0:.1f}s", flush=True)
    store["index"] = np.array(json.dumps(index))
    np.savez_compressed(os.path.join(HERE, "configs.npz"), **store)


if __name__ == "__main__":
    what = sys.argv[1:] or ["small", "configs"]
    if "small" in what:
        small_cases()
    if "configs" in what:
        config_cases()
