"""CPU tests of the product: C-ABI library, host LP, host-side API logic.

No GPU here: device entry points must refuse to run (there is no CPU
fallback), everything host-side must match the reference bit for bit.
"""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2506_00976_b200 as G
from conftest import ROOT, gpu_available
from oracle import port as P
from paper_2506_00976_b200 import _native


def _header_symbols():
    text = open(os.path.join(ROOT, "include", "gridot_b200.h")).read()
    return sorted(set(re.findall(r"\b(gdt_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(_native.LIB_PATH)
    syms = _header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_native.exported_symbols())
    assert b"sm_100a" in _native.lib().gdt_version()


def test_library_is_sm100a_cubin():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_c_abi_rejects_bad_arguments_without_touching_the_device():
    lib = _native.lib()
    dims = _native.i64s([6, 6])
    # dims not divisible by kappa -> GDT_ERR_ARG, no launch
    assert lib.gdt_sumpool_f64(None, None, 1, 2, dims, 4, None) == -1
    assert b"multiples of kappa" in lib.gdt_last_error()
    assert lib.gdt_interpolate(None, None, 1, 5, dims, dims, None, 0, None) == -1


@pytest.mark.parametrize("shape", [(1, 1), (1, 5), (5, 1), (7, 9), (30, 30)])
def test_native_simplex_matches_oracle_random(shape):
    rng = np.random.default_rng(sum(shape))
    for _ in range(5):
        C = rng.integers(0, 20, shape).astype(np.float64)  # many ties / degeneracy
        s = rng.random(shape[0]) + 0.01
        t = rng.random(shape[1]) + 0.01
        s /= s.sum()
        t /= t.sum()
        prob = G.build_transport_problem(s, t, C)
        cp, du, val = G.solve_transport(prob)
        st, bi, bj, bf, u, v, piv = P.simplex(prob.cost, prob.supply, prob.demand)
        keep = bf > 0
        assert np.array_equal(cp.row, bi[keep]) and np.array_equal(cp.col, bj[keep])
        assert cp.mass.tobytes() == bf[keep].tobytes()
        assert du.f.tobytes() == u.tobytes() and du.g.tobytes() == v.tobytes()


def test_native_simplex_matches_reference_plans(small_cases, config_cases):
    """Coarse C-tilde plans: support, flows and duals bit-exact vs the reference."""
    for c in list(small_cases) + [x for x in config_cases if "plan_row" in x]:
        dims, k, p = c["dims"], c["kappa"], c["p"]
        if "mu" in c:
            mc, nc = P.sumpool(c["mu"], dims, k), P.sumpool(c["nu"], dims, k)
        else:
            mc, nc = c["sumpool_mu"], c["sumpool_nu"]
        prob = G.build_transport_problem(mc, nc, P.centre_cost(dims, k, p))
        cp, du, _ = G.solve_transport(prob)
        assert np.array_equal(prob.src_index[cp.row], c["plan_row"]), c["tag"]
        assert np.array_equal(prob.dst_index[cp.col], c["plan_col"]), c["tag"]
        assert cp.mass.tobytes() == np.asarray(c["plan_mass"]).tobytes(), c["tag"]
        assert du.g.tobytes() == np.asarray(c["plan_v"]).tobytes(), c["tag"]


def test_solve_many_equals_single():
    rng = np.random.default_rng(9)
    probs = []
    for n in (3, 17, 40, 64):
        C = rng.random((n, n + 3))
        s, t = rng.random(n), rng.random(n + 3)
        probs.append(G.build_transport_problem(s / s.sum(), t / t.sum(), C))
    many = G.solve_transport_many(probs, threads=3)
    for prob, got in zip(probs, many):
        cp, du, val = G.solve_transport(prob)
        assert got[2] == val and got[0].mass.tobytes() == cp.mass.tobytes()


def test_warm_basis_matches_chained_and_cold():
    """A caller-supplied start basis (warm_basis) reproduces the in-call warm
    chain bit for bit, and both reach the cold solve's optimal value."""
    rng = np.random.default_rng(4)
    n = 48
    s, t = rng.random(n), rng.random(n)
    s, t = s / s.sum(), t / t.sum()
    t[np.argmax(t)] += s.sum() - t.sum()
    A, B = rng.random((n, n)), rng.random((n, n))
    pa, pb = (G.build_transport_problem(s, t, C) for C in (A, B))
    (first,), (basis,) = G.solve_transport_many([pa], threads=1, return_basis=True)
    chained = G.solve_transport_many([pa, pb], threads=1, warm_from=[-1, 0])[1]
    supplied = G.solve_transport_many([pb], threads=1, warm_basis=[basis])[0]
    cold = G.solve_transport(pb)
    assert supplied[2] == chained[2]
    assert supplied[0].mass.tobytes() == chained[0].mass.tobytes()
    assert abs(supplied[2] - cold[2]) <= 1e-12 * abs(cold[2])
    with pytest.raises(ValueError):
        G.solve_transport_many([pb], warm_basis=[(basis[0][:3], basis[1][:3], basis[2][:3])])


def test_lp_batch_hold_release_and_done_flags():
    """LPBatch: held jobs wait for release (issued from another thread while the
    native batch runs), chained jobs follow their parent, `finished` flags
    turn on as jobs complete, and results equal a plain batch's."""
    import threading
    import time

    rng = np.random.default_rng(11)
    n = 40
    s, t = rng.random(n), rng.random(n)
    s, t = s / s.sum(), t / t.sum()
    t[np.argmax(t)] += s.sum() - t.sum()
    C1 = rng.random((n, n))
    C2 = np.zeros((n, n))  # filled only after the batch has started
    probs = [G.build_transport_problem(s, t, C1), G.build_transport_problem(s, t, C2),
             G.build_transport_problem(s, t, C1)]
    batch = G.LPBatch(probs, warm_from=[-1, 0, 1], hold=[1])
    worker = threading.Thread(target=batch.run, kwargs={"threads": 2})
    worker.start()
    deadline = time.time() + 30
    while not batch.finished(0) and time.time() < deadline:
        time.sleep(0.001)
    assert batch.finished(0) and not batch.finished(1)
    C2[:] = rng.random((n, n))  # the held job's cost data arrives
    batch.release([1])
    worker.join(30)
    assert not worker.is_alive() and all(batch.finished(q) for q in range(3))
    ref = G.solve_transport_many([probs[0], G.build_transport_problem(s, t, C2.copy())],
                                 threads=1, warm_from=[-1, 0])
    assert batch.result(0)[2] == ref[0][2] and batch.result(1)[2] == ref[1][2]
    assert abs(batch.result(2)[2] - ref[0][2]) <= 1e-12 * abs(ref[0][2])


def test_lp_error_mapping():
    with pytest.raises(G.UnbalancedError):
        G.build_transport_problem(np.array([0.5, 0.5]), np.array([0.9]), np.ones((2, 1)))
    rng = np.random.default_rng(2)
    C = rng.random((12, 12))
    s = rng.random(12)
    prob = G.build_transport_problem(s / s.sum(), s[::-1] / s.sum(), C)
    with pytest.raises(G.IterationLimitError):
        G.solve_transport(prob, max_pivots=1)
    with pytest.raises(G.GridotError):
        G.build_transport_problem(np.zeros(3), np.ones(3) / 3, np.ones((3, 3)))


def test_data_model_validation():
    with pytest.raises(G.DimensionMismatchError):
        G.GridSpec(())
    with pytest.raises(G.DimensionMismatchError):
        G.GridSpec((3, 0))
    with pytest.raises(G.NegativeMassError) as ei:
        G.GridMeasure(G.GridSpec((3,)), np.array([0.1, -0.2, 0.3]))
    assert ei.value.index == 1
    with pytest.raises(ValueError):
        G.GridMeasure(G.GridSpec((2,)), np.array([np.nan, 1.0]))
    with pytest.raises(G.ZeroTotalMassError):
        G.normalize(G.GridMeasure(G.GridSpec((2,)), np.zeros(2)))
    with pytest.raises(ValueError):
        G.CoarseningSpec(0)
    spec = G.CoarseningSpec(4)
    assert spec.padded_dims(G.GridSpec((5, 8))) == (8, 8)
    assert spec.coarse_dims(G.GridSpec((5, 8))) == (2, 2)
    X = G.GridSpec((3, 2)).coordinates()
    assert X.tolist() == [[1, 1], [2, 1], [3, 1], [1, 2], [2, 2], [3, 2]]


def test_host_helpers_match_oracle():
    for dims, k, p in (((8, 8), 2, 2.0), ((6, 4, 4), 2, 1.0), ((12,), 3, 1.5)):
        grid, spec = G.GridSpec(dims), G.CoarseningSpec(k)
        assert G.min_cost_matrix(grid, spec, p).values.tobytes() == P.min_cost(dims, k, p).tobytes()
        c = G.coarsen_grid(grid, spec)
        assert c.tobytes() == P.block_centres(dims, k).tobytes()
        assert G.center_cost_matrix(c, c, p).values.tobytes() == \
            P.centre_cost(dims, k, p).tobytes()
        assert np.array_equal(G.block_index_map(grid, spec), P.block_ids(dims, k))
        assert G.tv_weights(grid, p).tobytes() == P.tv_weights(dims, p).tobytes()


def test_upscale_kernel_and_coupling_kats():
    """Known answers of test_bounds.py:61-157, re-expressed on this API."""
    k = G.UpscaleKernel.uniform(2, 1)
    assert np.allclose(k.weights, 0.25)
    k2 = G.UpscaleKernel(2, 1, np.array([[2.0, 0.0], [1.0, 1.0]]))
    assert np.allclose(k2.weights, [[0.5, 0.0], [0.25, 0.25]])
    with pytest.raises(ValueError):
        G.UpscaleKernel(2, 1, np.zeros((2, 2)))
    with pytest.raises(G.DimensionMismatchError):
        G.UpscaleKernel(2, 1, np.ones((2, 3)))
    coarse = G.SparseCoupling(np.array([0]), np.array([0]), np.array([1.0]), (1, 1))
    fine = G.upscale_coupling(coarse, G.UpscaleKernel.uniform(2, 1), (2,))
    assert sorted(zip(fine.row.tolist(), fine.col.tolist(), fine.mass.tolist())) == \
        [(0, 0, 0.25), (0, 1, 0.25), (1, 0, 0.25), (1, 1, 0.25)]
    rng = np.random.default_rng(4)
    raw = rng.random((2, 2, 2, 2)) + 0.01
    ker = G.UpscaleKernel(2, 2, raw)
    row, col = np.array([0, 1, 3]), np.array([2, 2, 0])
    m = rng.random(3)
    m /= m.sum()
    fine = G.upscale_coupling(G.SparseCoupling(row, col, m, (4, 4)), ker, (4, 4))
    blocks = G.block_index_map(G.GridSpec((4, 4)), G.CoarseningSpec(2))
    grouped = np.zeros((4, 4))
    np.add.at(grouped, (blocks[fine.row], blocks[fine.col]), fine.mass)
    dense = np.zeros((4, 4))
    dense[row, col] = m
    assert np.allclose(grouped, dense, atol=1e-12)
    with pytest.raises(G.DimensionMismatchError):
        G.upscale_coupling(coarse, G.UpscaleKernel.uniform(2, 1), (3,))


def test_reports_contract():
    assert G.signed_root(-8.0, 3.0) == -2.0
    assert G.signed_root(9.0, 2.0) == 3.0
    with pytest.raises(ValueError):
        G.BoundReport("x", float("inf"), 0.0)


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU behaviour")
def test_device_paths_fail_loudly_without_gpu():
    from paper_2506_00976_b200.device import NoDeviceError

    grid = G.GridSpec((4, 4))
    mu = G.GridMeasure(grid, np.full(16, 1 / 16))
    with pytest.raises(NoDeviceError):
        G.coarsen_measure(mu, G.CoarseningSpec(2))
    with pytest.raises(NoDeviceError):
        G.weighted_cost_upper_bound(mu, mu, 2, 2.0)
    with pytest.raises(NoDeviceError):
        G.quantized_bounds(mu.mass[None], mu.mass[None], (4, 4), 2, 2.0)


def test_exact_module_helpers():
    """grid_transport_problem / wasserstein_1d / hungarian_oracle (reference
    exact.py:139-253): the closed form and the assignment oracle agree with the
    host simplex on the same instances."""
    rng = np.random.default_rng(21)
    for n, p in ((12, 1.0), (12, 2.0), (9, 1.5)):
        a, b = rng.random(n), rng.random(n)
        ga = G.GridMeasure(G.GridSpec((n,)), a / a.sum())
        gb = G.GridMeasure(G.GridSpec((n,)), b / b.sum())
        lp = G.solve_transport(G.grid_transport_problem(ga, gb, p))[2] ** (1.0 / p)
        assert abs(G.wasserstein_1d(ga, gb, p) - lp) <= 1e-12 * lp
    k, l = np.array([2, 1, 3, 0, 2.0]), np.array([1, 1, 2, 3, 1.0])
    grid = G.GridSpec((5,))
    prob = G.grid_transport_problem(G.GridMeasure(grid, k / 8), G.GridMeasure(grid, l / 8), 2.0)
    assert G.hungarian_oracle(prob, 8) == 0.625
    assert abs(G.solve_transport(prob)[2] - 0.625) <= 1e-15
    with pytest.raises(G.QuantizationResidualError):
        G.hungarian_oracle(prob, 3)
    with pytest.raises(G.DimensionMismatchError):
        m2 = G.GridMeasure(G.GridSpec((2, 2)), np.full(4, 0.25))
        G.wasserstein_1d(m2, m2, 1.0)


def test_torch_extension_loads_the_c_abi():
    """The C library is loaded through the PyTorch extension (its linked
    dependency): torch.ops.gridot_b200 exists, calls into the same library,
    and its device operators are registered for CUDA tensors."""
    import torch

    _native.lib()
    ops = _native.torch_ops()
    assert ops is not None
    assert ops.version() == _native.lib().gdt_version().decode()
    for name in ("sumpool", "weighted_cost"):
        assert hasattr(ops, name)
    assert torch._C._dispatch_has_kernel_for_dispatch_key("gridot_b200::sumpool", "CUDA")
