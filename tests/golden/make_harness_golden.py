"""Golden CSV of the reference's bench matrix (build container only).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_harness_golden.py

Runs the LIVE reference ``gridot.cli.bench_run`` on a small matrix (all three
generator classes, exact + the four quantization bounds; exact + the two
entropic bounds) and writes ``tests/golden/harness_bench.csv``,
``tests/golden/harness_bench_reg.csv`` plus the generated measures of every pair
(``tests/golden/harness_measures.npz``), so ``paper_2506_00976_b200.harness``
can be checked for the same measures (CPU) and the same rows (GPU).
"""

from __future__ import annotations

import contextlib
import io
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.environ.get("GRIDOT_REF", "/root/reference/pkg/src"))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import gridot as G  # noqa: E402
from gridot import cli  # noqa: E402

CFG = dict(classes=("gaussians", "shapes", "noise"), n=8, d=2, p_values=(1.0, 2.0),
           kappas=(2, 4), seed=7, n_pairs=2,
           methods=("exact", "weighted_cost", "min_cost", "primal_upscaling", "dual_upscaling"))


def main():
    cfg = cli.BenchConfig(**CFG)
    rows = cli.bench_run(cfg)
    with open(os.path.join(HERE, "harness_bench.csv"), "w", newline="") as fh:
        cli.write_csv(rows, fh)
    meas = {}
    for ci, cls in enumerate(cfg.classes):
        for pi in range(cfg.n_pairs):
            for side in (0, 1):
                m = cli.gen_synthetic(cls, cfg.n, cfg.d, seed=[cfg.seed, ci, pi, side])
                meas[f"{cls}_{pi}_{side}"] = m.mass
    # a 3-D case for the generator only
    for cls in cfg.classes:
        meas[f"{cls}_3d"] = cli.gen_synthetic(cls, 6, 3, seed=[11, 2]).mass
    np.savez_compressed(os.path.join(HERE, "harness_measures.npz"), **meas)
    print(len(rows), "rows")
    # the entropic methods at the reference's default eps multipliers
    rcfg = cli.BenchConfig(**{**CFG, "n_pairs": 1,
                              "methods": ("exact", "reg_lower", "reg_upper")})
    rrows = cli.bench_run(rcfg)
    with open(os.path.join(HERE, "harness_bench_reg.csv"), "w", newline="") as fh:
        cli.write_csv(rrows, fh)
    print(len(rrows), "entropic rows")
    # the dist sub-command on two GRID files (every method, p in {1, 2})
    a = cli.gen_synthetic("gaussians", 8, 2, seed=[5, 0])
    b = cli.gen_synthetic("shapes", 8, 2, seed=[5, 1])
    c = cli.gen_synthetic("noise", 6, 2, seed=[5, 2])
    texts = {"a": G.dump_grid_measure(a), "b": G.dump_grid_measure(b),
             "c": G.dump_grid_measure(c)}
    cases = []
    with tempfile.TemporaryDirectory() as td:
        paths = {}
        for key, text in texts.items():
            paths[key] = os.path.join(td, key + ".grid")
            with open(paths[key], "w") as fh:
                fh.write(text)
        runs = [("a", "b", m, p, ["--kappa", "2"]) for p in ("1", "2")
                for m in ("exact", "weighted_cost", "min_cost", "primal_upscaling",
                          "dual_upscaling")]
        runs += [("a", "b", m, "2", ["--eps", "0.004"]) for m in ("reg_lower", "reg_upper")]
        runs += [("a", "c", "exact", "2", []), ("a", "b", "nope", "2", [])]
        for mu, nu, m, p, extra in runs:
            out, err = io.StringIO(), io.StringIO()
            with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
                rc = cli.main(["dist", "--mu", paths[mu], "--nu", paths[nu], "--method", m,
                               "--p", p] + extra)
            cases.append({"mu": mu, "nu": nu, "method": m, "p": p, "extra": extra, "rc": rc,
                          "stdout": out.getvalue()})
    with open(os.path.join(HERE, "harness_dist.json"), "w") as fh:
        json.dump({"grids": texts, "cases": cases}, fh, indent=0)
    print(len(cases), "dist cases")


if __name__ == "__main__":
    main()
