"""Entropic-bound fixtures from the LIVE reference (build container only).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_entropic_golden.py

Runs the reference's ``reg_lower_bound`` / ``reg_upper_bound``
(sinkhorn.py:226-299) on seeded grid pairs -- Dirac pairs, identical
measures, holes in the supports, iteration caps, epsilons small enough that
the plain kernel underflows and the log-domain restart runs, 1-D to 3-D,
p in {1, 1.5, 2} -- and writes ``tests/golden/entropic.npz``: inputs, every
report field, and whether the log domain ran.
"""

from __future__ import annotations

import json
import logging
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.environ.get("GRIDOT_REF", "/root/reference/pkg/src"))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import gridot as G  # noqa: E402


class _Catch(logging.Handler):
    def __init__(self):
        super().__init__()
        self.hit = False

    def emit(self, record):
        if "log domain" in record.getMessage():
            self.hit = True


def _pair(rng, dims, holes=0.0):
    n = int(np.prod(dims))
    a, b = rng.random(n), rng.random(n)
    if holes:
        a[rng.random(n) < holes] = 0.0
        b[rng.random(n) < holes] = 0.0
    return a / a.sum(), b / b.sum()


def cases():
    rng = np.random.default_rng(777)
    out = []
    d2 = (np.array([1.0, 0.0]), np.array([0.0, 1.0]))
    for eps in (0.5, 0.1, 1e-3):
        out.append(("dirac", (2,), *d2, 1.0, eps, 1e-9, 10_000))
    m = rng.random(9)
    m /= m.sum()
    out.append(("identical", (3, 3), m, m.copy(), 2.0, 2.0, 1e-9, 10_000))
    for k in range(6):
        p = (1.0, 2.0)[k % 2]
        eps = (0.1, 1.0, 5.0)[k % 3]
        out.append((f"line{k}", (6,), *_pair(rng, (6,)), p, eps, 1e-9, 10_000))
    pr = _pair(rng, (4, 4))
    for cap in (1, 2, 5):
        out.append((f"cap{cap}", (4, 4), *pr, 2.0, 5.0, 1e-12, cap))
    out.append(("logdom4x4", (4, 4), *pr, 2.0, 0.05, 1e-9, 5000))
    out.append(("g8p2", (8, 8), *_pair(rng, (8, 8)), 2.0, 0.5 * 64, None, 10_000))
    out.append(("g8p1", (8, 8), *_pair(rng, (8, 8)), 1.0, 0.5 * 8, None, 10_000))
    out.append(("g12x10holes", (12, 10), *_pair(rng, (12, 10), 0.25), 2.0, 0.1 * 144, None, 10_000))
    out.append(("g16p15", (16, 16), *_pair(rng, (16, 16)), 1.5, 0.1 * 16 ** 1.5, None, 10_000))
    out.append(("g5x4x3", (5, 4, 3), *_pair(rng, (5, 4, 3)), 2.0, 2.0, 1e-10, 10_000))
    out.append(("g32p2", (32, 32), *_pair(rng, (32, 32)), 2.0, 0.05 * 1024, None, 10_000))
    out.append(("g24log", (24, 24), *_pair(rng, (24, 24), 0.1), 2.0, 0.4, 1e-8, 300))
    out.append(("g20p1cap", (20, 20), *_pair(rng, (20, 20)), 1.0, 0.2, 1e-12, 40))
    out.append(("g16holes_tiny", (16, 16), *_pair(rng, (16, 16), 0.3), 2.0, 0.01, 1e-9, 200))
    a, b = _pair(rng, (10, 10))
    a = a.reshape(10, 10, order="F")
    b = b.reshape(10, 10, order="F")
    a[5:, :] = 0.0
    b[:5, :] = 0.0
    out.append(("g10split", (10, 10), (a / a.sum()).ravel(order="F"),
                (b / b.sum()).ravel(order="F"), 2.0, 0.05, 1e-9, 300))
    out.append(("g12holes_p1", (12, 12), _pair(rng, (12, 12))[0], _pair(rng, (12, 12), 0.5)[1],
                1.0, 0.004, 1e-9, 150))
    return out


def main():
    h = _Catch()
    lg = logging.getLogger("gridot.sinkhorn")
    lg.addHandler(h)
    lg.setLevel(logging.INFO)
    rec = {}
    meta = []
    for q, (tag, dims, mu, nu, p, eps, xi, mi) in enumerate(cases()):
        grid = G.GridSpec(dims)
        m1, m2 = G.GridMeasure(grid, mu), G.GridMeasure(grid, nu)
        X = grid.coordinates()
        cost = G.CostSpec(X, X, p)
        params = G.RegularizationParams(eps, xi=xi, max_iter=mi)
        h.hit = False
        lo = G.reg_lower_bound(m1, m2, cost, params)
        log_lo = h.hit
        h.hit = False
        up = G.reg_upper_bound(m1, m2, cost, params)
        rec[f"c{q}_mu"], rec[f"c{q}_nu"] = mu, nu
        meta.append({"tag": tag, "dims": list(dims), "p": p, "eps": eps, "xi": xi,
                     "max_iter": mi, "log_domain": bool(log_lo),
                     "lower": {"value": lo.value, "raw_value": lo.raw_value,
                               "iterations": lo.iterations, **lo.components},
                     "upper": {"value": up.value, "raw_value": up.raw_value,
                               "iterations": up.iterations, **up.components}})
        print(tag, lo.value, up.value, lo.iterations, "log" if log_lo else "")
    rec["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(HERE, "entropic.npz"), **rec)


if __name__ == "__main__":
    main()
