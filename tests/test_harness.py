"""Bench-matrix harness (reference cli.py bench): generators, config checks,
CSV schema and the exact baseline on CPU; the full device matrix against the
reference's own CSV on the GPU (tests/golden/make_harness_golden.py)."""

from __future__ import annotations

import csv
import io
import json
import os

import numpy as np
import pytest

from paper_2506_00976_b200 import harness as H

GOLD = os.path.join(os.path.dirname(__file__), "golden")
CFG = dict(classes=("gaussians", "shapes", "noise"), n=8, d=2, p_values=(1.0, 2.0),
           kappas=(2, 4), seed=7, n_pairs=2,
           methods=("exact", "weighted_cost", "min_cost", "primal_upscaling", "dual_upscaling"))


def _golden_rows():
    with open(os.path.join(GOLD, "harness_bench.csv")) as fh:
        return list(csv.DictReader(fh))


def test_generators_match_reference_bit_for_bit():
    z = np.load(os.path.join(GOLD, "harness_measures.npz"))
    for ci, cls in enumerate(CFG["classes"]):
        for pi in range(CFG["n_pairs"]):
            for side in (0, 1):
                m = H.gen_synthetic(cls, 8, 2, seed=[7, ci, pi, side])
                assert np.array_equal(m.mass, z[f"{cls}_{pi}_{side}"]), (cls, pi, side)
        assert np.array_equal(H.gen_synthetic(cls, 6, 3, seed=[11, 2]).mass, z[f"{cls}_3d"])


def test_config_validation_and_schema():
    H.BenchConfig(**CFG).validate()
    for bad in (dict(n=3), dict(d=0), dict(n=300), dict(p_values=(0.5,)), dict(kappas=(0,)),
                dict(xi=0.0), dict(n_pairs=0), dict(methods=()), dict(eps_multipliers=(0.0,)),
                dict(methods=("nope",)), dict(max_iter=0), dict(precision="bf16"),
                dict(classes=("blobs",))):
        with pytest.raises(H.CliValidationError):
            H.BenchConfig(**{**CFG, **bad}).validate()
    with pytest.raises(H.CliValidationError):
        H.gen_synthetic("gaussians", 3, 2, 0)
    row = H.ReportRow("x-000", "min_cost", 2.0, "4", bound=1.0 / 3.0, exact=None)
    assert row.as_record() == ["x-000", "min_cost", "2", "4", "0.33333333333333331", "", "",
                               "", "", ""]
    text = H.rows_to_csv([row])
    assert text.splitlines()[0] == ",".join(H.CSV_COLUMNS)
    assert H._relative_error("min_cost", 1.0, 2.0) == 0.5
    assert H._relative_error("weighted_cost", 3.0, 2.0) == 0.5
    assert H.main(["bench", "--methods", "reg_upper", "--eps", "0"]) == 1
    H.BenchConfig(**{**CFG, "methods": ("reg_lower", "reg_upper")}).validate()


def test_exact_baseline_matches_reference():
    gold = {(r["pair"], float(r["p"])): float(r["exact"]) for r in _golden_rows()
            if r["method"] == "exact"}
    for ci, cls in enumerate(CFG["classes"]):
        mus = [H.gen_synthetic(cls, 8, 2, seed=[7, ci, i, 0]).mass for i in range(2)]
        nus = [H.gen_synthetic(cls, 8, 2, seed=[7, ci, i, 1]).mass for i in range(2)]
        for p in CFG["p_values"]:
            out = H.exact_distances(mus, nus, 8, 2, p, threads=1)
            for i, (value, wall, err) in enumerate(out):
                assert err == ""
                ref = gold[(f"{cls}-{i:03d}", p)]
                assert abs(value - ref) <= 1e-15 * ref, (cls, i, p, value, ref)


@pytest.mark.gpu
def test_device_bench_matrix_matches_reference_csv():
    rows = H.bench_run(H.BenchConfig(**CFG))
    gold = _golden_rows()
    assert len(rows) == len(gold)
    got = list(csv.DictReader(io.StringIO(H.rows_to_csv(rows))))
    for g, r in zip(gold, got):
        assert (g["pair"], g["method"], g["p"], g["param"]) == \
            (r["pair"], r["method"], r["p"], r["param"])
        assert bool(g["error"]) == bool(r["error"]), (g, r)
        if g["error"]:
            assert g["error"].split(":")[0] == r["error"].split(":")[0]
            continue
        for key in ("bound", "exact", "rel_error"):
            a, b = float(g[key]), float(r[key])
            assert abs(a - b) <= 1e-9 * max(1.0, abs(a)), (g["pair"], g["method"], key, a, b)


@pytest.mark.gpu
def test_device_entropic_rows_match_reference_csv():
    """reg_lower / reg_upper rows at the reference's default eps multipliers
    (cli.py:123, epsilon = multiplier * n^p).  The lower bound is a dual value
    (1e-9); the upper bound carries weighted-TV corrections whose rounding
    noise the 1/p root amplifies (tests/test_entropic.py), hence 1e-7."""
    with open(os.path.join(GOLD, "harness_bench_reg.csv")) as fh:
        gold = list(csv.DictReader(fh))
    cfg = H.BenchConfig(**{**CFG, "n_pairs": 1, "methods": ("exact", "reg_lower", "reg_upper")})
    got = list(csv.DictReader(io.StringIO(H.rows_to_csv(H.bench_run(cfg)))))
    assert len(got) == len(gold)
    for g, r in zip(gold, got):
        assert (g["pair"], g["method"], g["p"], g["param"]) == \
            (r["pair"], r["method"], r["p"], r["param"])
        assert bool(g["error"]) == bool(r["error"]), (g, r)
        if g["error"]:
            continue
        tol = 1e-7 if g["method"] == "reg_upper" else 1e-9
        a, b = float(g["bound"]), float(r["bound"])
        assert abs(a - b) <= tol * max(1.0, abs(a)), (g["pair"], g["method"], g["param"], a, b)


DIST = json.load(open(os.path.join(GOLD, "harness_dist.json")))


def _dist_cases(gpu: bool):
    out = []
    for c in DIST["cases"]:
        needs_gpu = c["method"] not in ("exact", "nope")
        if needs_gpu == gpu:
            out.append(c)
    return out


def _run_dist(tmp_path, c, capsys):
    paths = {}
    for key, text in DIST["grids"].items():
        paths[key] = tmp_path / f"{key}.grid"
        paths[key].write_text(text)
    rc = H.main(["dist", "--mu", str(paths[c["mu"]]), "--nu", str(paths[c["nu"]]),
                 "--method", c["method"], "--p", c["p"]] + c["extra"])
    return rc, capsys.readouterr().out


def _same_record(got: str, want: str, tol: float):
    g, w = got.strip().split(","), want.strip().split(",")
    assert len(g) == len(w) == len(H.CSV_COLUMNS)
    assert g[:4] == w[:4] and g[9] == w[9]
    for i in (4, 5, 6):  # bound, exact, rel_error
        assert (g[i] == "") == (w[i] == "")
        if w[i]:
            assert abs(float(g[i]) - float(w[i])) <= tol * max(1.0, abs(float(w[i]))), (i, g, w)


@pytest.mark.parametrize("c", _dist_cases(False), ids=lambda c: f"{c['method']}-{c['nu']}")
def test_dist_host_methods_match_reference(tmp_path, capsys, c):
    """`dist` (cli.py:358-445) with the host methods: the exact LP value bit for
    bit, and the reference's exit codes for bad arguments / mismatched grids."""
    rc, out = _run_dist(tmp_path, c, capsys)
    assert rc == c["rc"]
    if c["rc"] == 0:
        _same_record(out, c["stdout"], 0.0)


@pytest.mark.gpu
@pytest.mark.parametrize("c", _dist_cases(True), ids=lambda c: f"{c['method']}-p{c['p']}")
def test_dist_device_methods_match_reference(tmp_path, capsys, c):
    rc, out = _run_dist(tmp_path, c, capsys)
    assert rc == c["rc"]
    _same_record(out, c["stdout"], 1e-7 if c["method"] == "reg_upper" else 1e-9)
