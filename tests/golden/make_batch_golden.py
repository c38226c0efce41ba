"""Reference values for EVERY pair the benchmark times (build container only).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_batch_golden.py [cfg ...] [--workers 8]

Runs the LIVE reference (``gridot``'s four bound functions, quantized.py:172,
199, 288, 487, as ``cli._pair_rows`` calls them, cli.py:247-270) on the
benched batches of the BASELINE configurations and writes
``tests/golden/batch_cfg{c}.npz``:

* cfg2 pairs 0-44, cfg3 pairs 0-44 x 4 (kappa, p), cfg4 pairs 0-44 (one GPU's
  shard of the 360-pair job), cfg5 pairs 0-63 — exactly what ``bench.py``
  times on one GPU;
* per pair and combination: every raw bound value and component, the IPF
  iteration count, and SHA-256 digests of the reference's coarse C-tilde plan
  (basic arcs with flow > 0 in the reference's order: full coarse row ids,
  column ids, masses; and the dual vector g) plus its arc count;
* SHA-256 of the generated masses, so the fixture pins the generator too.

Inputs are regenerated from seeds by ``paper_2506_00976_b200.synthetic``; the
reference never travels to the GPU box, these values do.
"""

from __future__ import annotations

import hashlib
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
REF = os.environ.get("GRIDOT_REF", "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

BATCH = {2: 45, 3: 45, 4: 45, 5: 64}
FIELDS = ("wc_value", "mc_raw", "pu_value", "pu_transport", "pu_delta_mu", "pu_delta_nu",
          "pu_marginal_gap", "pu_converged", "pu_iterations", "du_raw", "du_dual_value",
          "plan_arcs", "seconds")


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def one(task):
    cfg, pair, kappa, p = task
    sys.path.insert(0, REF)
    import gridot as G
    from gridot.quantized import _solve_coarse_center

    from paper_2506_00976_b200 import synthetic as S

    wl = S.WORKLOADS[cfg]
    mu, nu = S.measure(cfg, pair, 0), S.measure(cfg, pair, 1)
    t0 = time.perf_counter()
    grid = G.GridSpec(wl.dims)
    gm, gn = G.GridMeasure(grid, mu), G.GridMeasure(grid, nu)
    wc = G.weighted_cost_upper_bound(gm, gn, kappa, p)
    mc = G.min_cost_lower_bound(gm, gn, kappa, p)
    pu = G.primal_upscaling_upper_bound(gm, gn, kappa, p, xi=wl.xi, max_iter=wl.max_iter)
    du = G.dual_upscaling_lower_bound(gm, gn, kappa, p)
    secs = time.perf_counter() - t0
    full, _problem, duals, _, _, _ = _solve_coarse_center(gm, gn, G.CoarseningSpec(kappa), p)
    rec = {
        "wc_value": wc.value, "mc_raw": mc.raw_value, "pu_value": pu.value,
        "pu_transport": pu.components["transport"], "pu_delta_mu": pu.components["delta_mu"],
        "pu_delta_nu": pu.components["delta_nu"],
        "pu_marginal_gap": pu.components["marginal_gap"],
        "pu_converged": pu.components["converged"], "pu_iterations": float(pu.iterations),
        "du_raw": du.raw_value, "du_dual_value": du.components["dual_value"],
        "plan_arcs": float(len(full.row)), "seconds": secs,
    }
    plan = digest(np.asarray(full.row, np.int64), np.asarray(full.col, np.int64),
                  np.asarray(full.mass, np.float64))
    dual = digest(np.asarray(duals.g, np.float64))
    return task, rec, plan, dual, digest(mu.astype(np.float64)), digest(nu.astype(np.float64))


def main(argv):
    workers = 8
    if "--workers" in argv:
        i = argv.index("--workers")
        workers = int(argv[i + 1])
        argv = argv[:i] + argv[i + 2:]
    cfgs = [int(a) for a in argv] or [4, 5, 3, 2]
    from paper_2506_00976_b200 import synthetic as S

    tasks = []
    for cfg in cfgs:
        wl = S.WORKLOADS[cfg]
        for pair in range(BATCH[cfg]):
            for kappa, p in wl.combos:
                tasks.append((cfg, pair, int(kappa), float(p)))
    results = {}
    t0 = time.time()
    with mp.get_context("spawn").Pool(workers) as pool:
        for k, res in enumerate(pool.imap_unordered(one, tasks)):
            results[res[0]] = res
            if k % 20 == 0:
                print(f"{k + 1}/{len(tasks)} {time.time() - t0:.0f}s", flush=True)
    for cfg in cfgs:
        wl = S.WORKLOADS[cfg]
        combos = [(int(k), float(p)) for k, p in wl.combos]
        B = BATCH[cfg]
        vals = np.zeros((B, len(combos), len(FIELDS)))
        plans = np.empty((B, len(combos)), dtype="U64")
        duals = np.empty((B, len(combos)), dtype="U64")
        mu_sha = np.empty(B, dtype="U64")
        nu_sha = np.empty(B, dtype="U64")
        for b in range(B):
            for j, (k, p) in enumerate(combos):
                _, rec, pl, du, ms, ns = results[(cfg, b, k, p)]
                vals[b, j] = [rec[f] for f in FIELDS]
                plans[b, j], duals[b, j] = pl, du
                mu_sha[b], nu_sha[b] = ms, ns
        meta = {"cfg": cfg, "pairs": B, "combos": combos, "fields": list(FIELDS),
                "xi": wl.xi, "max_iter": wl.max_iter, "dims": list(wl.dims),
                "reference": "gridot (live, /root/reference/pkg/src)",
                "numpy": np.__version__}
        np.savez_compressed(os.path.join(HERE, f"batch_cfg{cfg}.npz"), values=vals,
                            plan_sha=plans, dual_sha=duals, mu_sha=mu_sha, nu_sha=nu_sha,
                            meta=np.array(json.dumps(meta)))
        print(f"cfg{cfg}: {B} pairs x {len(combos)} combos, reference "
              f"{vals[:, :, -1].sum():.0f} core-seconds", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
