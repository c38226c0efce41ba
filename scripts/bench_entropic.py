#!/usr/bin/env python
"""Entropic-bound throughput (reg_lower_bound path, sinkhorn.py:150-299).

Times gdt_entropic_fit on one GPU at fixed sweep counts (xi tiny) and reports
the per-sweep time from the difference of two runs (K fill excluded), the
algorithmic HBM traffic of a sweep (two passes over the dense fp64 kernel:
16 * ns * nt bytes) and the achieved fraction of the measured HBM peak; the
CPU oracle (numpy BLAS, all cores) is timed on the smallest grid.
One JSON line per grid.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2506_00976_b200 as G  # noqa: E402
from paper_2506_00976_b200 import _native as N  # noqa: E402
from paper_2506_00976_b200.device import stream, to_dev, torch  # noqa: E402


def peak_hbm():
    try:
        return float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(
            os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 7672.0


def fit_seconds(xs, xt, mu, nu, ns, nt, sweeps, scratch, f, g, info, st, p, eps):
    t = torch()
    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    t.cuda.synchronize()
    e0.record()
    N.check(N.lib().gdt_entropic_fit(N.ptr(xs), N.ptr(xt), ns, nt, xs.shape[1], p, eps,
                                     N.ptr(mu), N.ptr(nu), 1e-300, sweeps, N.ptr(f), N.ptr(g),
                                     N.ptr(info), N.ptr(st), N.ptr(scratch), stream()), "fit")
    e1.record()
    t.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3


def main():
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--sides", default="64,128,256")
    args = ap.parse_args()
    t = torch()
    from paper_2506_00976_b200.device import device

    device()
    for side in (int(x) for x in args.sides.split(",")):
        dims = (side, side)
        grid = G.GridSpec(dims)
        n = grid.cell_count
        rng = np.random.default_rng(side)
        mu, nu = rng.random(n) + 0.1, rng.random(n) + 0.1
        mu, nu = mu / mu.sum(), nu / nu.sum()
        X = grid.coordinates()
        p, eps = 2.0, 0.05 * side ** 2
        xs = to_dev(np.ascontiguousarray(X))
        mu_d, nu_d = to_dev(mu), to_dev(nu)
        scratch = t.empty(int(N.lib().gdt_entropic_scratch_bytes(n, n)), dtype=t.uint8,
                          device=mu_d.device)
        f = t.empty(n, dtype=t.float64, device=mu_d.device)
        g = t.empty(n, dtype=t.float64, device=mu_d.device)
        info = t.empty(4, dtype=t.float64, device=mu_d.device)
        st = t.empty(1, dtype=t.int32, device=mu_d.device)
        args = (xs, xs, mu_d, nu_d, n, n)
        fit_seconds(*args, 3, scratch, f, g, info, st, p, eps)  # warm-up
        s_lo, s_hi = 20, 60
        t_lo = min(fit_seconds(*args, s_lo, scratch, f, g, info, st, p, eps) for _ in range(2))
        t_hi = min(fit_seconds(*args, s_hi, scratch, f, g, info, st, p, eps) for _ in range(2))
        per = (t_hi - t_lo) / (s_hi - s_lo)
        bytes_sweep = 16.0 * n * n
        rec = {"workload": f"entropic fit {side}x{side} (ns = nt = {n}), p=2, fp64",
               "kernel_bytes": 8 * n * n, "sweep_ms": per * 1e3,
               "achieved_gbs": bytes_sweep / per / 1e9, "peak_gbs": peak_hbm(),
               "frac": bytes_sweep / per / 1e9 / peak_hbm(),
               "work": "16 * ns * nt bytes per sweep (two passes over the fp64 kernel)",
               "fit_ms_60_sweeps": t_hi * 1e3}
        if side == 64:
            from oracle import port as P  # CPU baseline only

            K = np.exp(-P.costs(X, X, p) / eps)
            t0 = time.perf_counter()
            P.ipf(K, mu, nu, 1e-300, 20)
            rec["cpu_oracle_sweep_ms"] = (time.perf_counter() - t0) / 20 * 1e3
            rec["cpu_cores"] = os.cpu_count()
        print(json.dumps(rec), flush=True)
        del scratch
        t.cuda.empty_cache()


if __name__ == "__main__":
    main()
