"""Parity on EXACTLY the batches bench.py times, against the live reference.

tests/golden/batch_cfg{2,3,4,5}.npz hold the reference's own results
(``gridot`` run by tests/golden/make_batch_golden.py in the build container)
for every pair one GPU benchmarks: cfg2 pairs 0-44, cfg3 pairs 0-44 x 4
(kappa, p), cfg4 pairs 0-44 (one GPU's shard of 360), cfg5 pairs 0-63.  Each
batch runs through the public batched API ``quantized_bounds_many`` -- the
call the e2e benchmark makes -- in both precisions, and every pair and
combination is checked:

* coarse C-tilde plan (basic arcs with flow > 0, their order, flows, and the
  dual vector g) bit-exact against the reference's, on the GPU SumPool path
  (the plans returned through ``plans_out`` are solved from the device's
  coarse masses);
* every raw bound value within the north-star tolerance: 1e-9 relative in
  fp64 mode, 1e-5 in fp32 mode (quantized.py:172-521 / cli.py:282-295);
* IPF iteration count equal to the reference's;
* lower <= upper on every pair and combination (kappa = 8 included).
"""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

G = pytest.importorskip("paper_2506_00976_b200")
from paper_2506_00976_b200 import synthetic as S  # noqa: E402


def load(cfg):
    z = np.load(os.path.join(GOLDEN, f"batch_cfg{cfg}.npz"), allow_pickle=False)
    meta = json.loads(str(z["meta"]))
    return z, meta


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def rel(a, b, floor=1e-300):
    return abs(a - b) / max(abs(a), abs(b), floor)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("cfg", [2, 3, 4, 5])
def test_benched_batch_matches_reference(cfg, precision):
    z, meta = load(cfg)
    wl = S.WORKLOADS[cfg]
    B = meta["pairs"]
    combos = [tuple(c) for c in meta["combos"]]
    F = {f: i for i, f in enumerate(meta["fields"])}
    vals = z["values"]
    mus, nus = S.batch(cfg, 0, B)
    plans = {}
    res = G.quantized_bounds_many(mus, nus, wl.dims, combos, precision=precision, xi=wl.xi,
                                  max_iter=wl.max_iter, return_exceptions=False,
                                  plans_out=plans)
    tol = 1e-9 if precision == "fp64" else 1e-5
    bad = []
    for j, (k, p) in enumerate(combos):
        key = (int(k), float(p))
        for b in range(B):
            ref = vals[b, j]
            rep = res[key][b]
            tag = f"cfg{cfg} pair {b} k{k} p{p:g} {precision}"
            rows, cols, mass, g, _ = plans[key][b]
            if digest(np.asarray(rows, np.int64), np.asarray(cols, np.int64),
                      np.asarray(mass, np.float64)) != str(z["plan_sha"][b, j]):
                bad.append(f"{tag}: C-tilde plan differs ({len(rows)} arcs, reference "
                           f"{int(ref[F['plan_arcs']])})")
            if digest(np.asarray(g, np.float64)) != str(z["dual_sha"][b, j]):
                bad.append(f"{tag}: C-tilde duals differ")
            pu = rep["primal_upscaling"]
            checks = [
                ("weighted_cost", rep["weighted_cost"].raw_value, ref[F["wc_value"]], tol),
                ("min_cost", rep["min_cost"].raw_value, ref[F["mc_raw"]], 1e-12),
                ("primal_upscaling", pu.value, ref[F["pu_value"]], tol),
                ("pu.transport", pu.components["transport"], ref[F["pu_transport"]], tol),
                ("dual_upscaling", rep["dual_upscaling"].raw_value, ref[F["du_raw"]], tol),
                ("du.dual_value", rep["dual_upscaling"].components["dual_value"],
                 ref[F["du_dual_value"]], tol),
            ]
            for name, got, want, t in checks:
                if rel(got, want) > t:
                    bad.append(f"{tag}: {name} {got!r} vs reference {want!r} "
                               f"(rel {rel(got, want):.2e} > {t:g})")
            # TV terms are rounding-level residuals of the marginals: absolute,
            # on the bound's own scale
            for name in ("delta_mu", "delta_nu"):
                got, want = pu.components[name], ref[F[f"pu_{name}"]]
                if abs(got - want) > tol * abs(ref[F["pu_value"]]):
                    bad.append(f"{tag}: pu.{name} {got!r} vs {want!r}")
            if pu.iterations != int(ref[F["pu_iterations"]]):
                bad.append(f"{tag}: IPF iterations {pu.iterations} vs "
                           f"{int(ref[F['pu_iterations']])}")
            if pu.components["converged"] != ref[F["pu_converged"]]:
                bad.append(f"{tag}: converged flag differs")
            lo = max(rep["min_cost"].value, rep["dual_upscaling"].value)
            hi = min(rep["weighted_cost"].value, pu.value)
            if not lo <= hi:
                bad.append(f"{tag}: bracket inverted {lo!r} > {hi!r}")
    assert not bad, f"{len(bad)} mismatches:\n" + "\n".join(bad[:40])
