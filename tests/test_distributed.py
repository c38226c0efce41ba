"""Multi-process host logic of the data-parallel path (gloo, world_size 2, CPU).

The device compute is per pair and has no collective; what crosses ranks is
the sharding and the all_gather of fixed-width records.  These tests run two
gloo ranks on 127.0.0.1 and check that gathering reproduces the single-rank
table bit for bit, including uneven shards and failed methods.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2506_00976_b200 import distributed as D
from paper_2506_00976_b200.errors import ZeroDenominatorError
from paper_2506_00976_b200.reports import BoundReport


def _fake_reports(lo, hi):
    out = []
    for i in range(lo, hi):
        rep = {
            "weighted_cost": BoundReport("weighted_cost", 10.0 + i, 10.0 + i,
                                         {"transport": 10.0 + i}, 0.5, None, 1024),
            "min_cost": BoundReport("min_cost", max(0.0, i - 3.0), i - 3.0,
                                    {"transport": i - 3.0}, 0.5, None, 1024),
            "dual_upscaling": BoundReport("dual_upscaling", 5.0 + i / 7, 5.0 + i / 7,
                                          {"dual_value": (5.0 + i / 7) ** 2}, 0.5, None, 1024),
        }
        if i % 3 == 2:
            rep["primal_upscaling"] = ZeroDenominatorError("ring fallback failed")
        else:
            rep["primal_upscaling"] = BoundReport(
                "primal_upscaling", 11.0 + i, 11.0 + i,
                {"transport": 11.0 + i - 1e-9, "delta_mu": 5e-10, "delta_nu": 5e-10,
                 "marginal_gap": 1e-16, "converged": 1.0}, 0.5, 1, 1024)
        out.append(rep)
    return out


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, total, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = D.shard_range(total, rank, world)
    local = D.pack_records(_fake_reports(lo, hi), lo)
    table = D.gather_records(local, total)
    q.put((rank, table))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [8, 7, 1])
def test_gloo_gather_matches_single_rank(total):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect = D.pack_records(_fake_reports(0, total), 0)
    for r in range(world):
        assert got[r].shape == expect.shape
        assert np.array_equal(got[r], expect, equal_nan=True)


COMBOS = ((4, 1.0), (4, 2.0), (8, 1.0))


def _fake_many(mus, nus, dims, combos, **kw):
    """Host stand-in for quantized_bounds_many: values depend on the pair's
    global index (mus[:, 0]) and the combination, so a misplaced row cannot
    go unnoticed."""
    out = {}
    for k, p in combos:
        rows = []
        for m in mus:
            i = int(m[0])
            rep = _fake_reports(i, i + 1)[0]
            rows.append({key: (BoundReport(r.method, r.value + k + p, r.raw_value + k + p,
                                           r.components, r.wall_time, r.iterations,
                                           r.coarse_size)
                               if isinstance(r, BoundReport) else r)
                         for key, r in rep.items()})
        out[(k, p)] = rows
    return out


def _many_worker(rank, world, port, total, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mus = np.arange(total, dtype=np.float64)[:, None] * np.ones((1, 4))
    _, table = D.distributed_bounds_many(mus, mus, (2, 2), COMBOS, compute=_fake_many)
    q.put((rank, table))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [7, 2, 1])
def test_gloo_distributed_bounds_many_matches_single_rank(total):
    """The multi-combination path: one compute call per rank on its shard,
    one all_gather of pair-major records, same table as one rank alone."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_many_worker, args=(r, world, port, total, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    mus = np.arange(total, dtype=np.float64)[:, None] * np.ones((1, 4))
    single = _fake_many(mus, mus, (2, 2), COMBOS)
    expect = np.stack([D.pack_records(single[key], 0) for key in COMBOS])
    for r in range(world):
        assert got[r].shape == (len(COMBOS), total, D.F)
        assert np.array_equal(got[r], expect, equal_nan=True)


def test_record_keeps_coarse_size_without_weighted_cost():
    reps = _fake_reports(0, 3)
    for rep in reps:
        del rep["weighted_cost"]
    back = D.unpack_records(D.pack_records(reps, 0))
    for b in back:
        for r in b["reports"].values():
            assert r.coarse_size == 1024 and r.wall_time == 0.5


def test_shard_range_partitions_exactly():
    for total in (0, 1, 7, 45, 360):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                lo, hi = D.shard_range(total, r, world)
                assert hi - lo in (total // world, -(-total // world))
                seen.extend(range(lo, hi))
            assert seen == list(range(total))


def test_pack_unpack_roundtrip():
    reps = _fake_reports(0, 6)
    back = D.unpack_records(D.pack_records(reps, 0))
    for i, (a, b) in enumerate(zip(reps, back)):
        assert b["pair"] == i
        for m in ("weighted_cost", "min_cost", "dual_upscaling"):
            assert b["reports"][m].raw_value == a[m].raw_value
            assert b["reports"][m].value == a[m].value
        if isinstance(a["primal_upscaling"], Exception):
            assert "primal_upscaling" not in b["reports"] and b["status"] & 4
        else:
            assert b["reports"]["primal_upscaling"].components == a["primal_upscaling"].components


def _bench_e2e_worker(rank, world, port, q):
    """bench.run_e2e under torchrun semantics (world 2, gloo), with a host
    stand-in for the device computation: sharding, the gather of records,
    the max-over-ranks time and the single-process check of the gathered table."""
    import argparse
    import sys

    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    from paper_2506_00976_b200 import synthetic as S

    def fake(mus, nus, dims, combos, **kw):
        mus = np.asarray(mus)
        out = {}
        for k, p in combos:
            rows = []
            for m in mus:
                v = float(m[0] * 1e6) + k + p
                pu = BoundReport("primal_upscaling", v, v,
                                 {"transport": v, "delta_mu": 0.0, "delta_nu": 0.0,
                                  "marginal_gap": 0.0, "converged": 1.0}, 0.1, 1, 64)
                du = BoundReport("dual_upscaling", v, v, {"dual_value": v * v}, 0.1, None, 64)
                wc = BoundReport("weighted_cost", v, v, {"transport": v}, 0.1, None, 64)
                rows.append({"weighted_cost": wc, "min_cost": wc, "primal_upscaling": pu,
                             "dual_upscaling": du})
            out[(int(k), float(p))] = rows
        return out

    class G:  # the public API the single-process check calls
        quantized_bounds_many = staticmethod(fake)

    D.quantized_bounds_many = fake  # the per-rank compute of distributed_bounds_many
    bench.CFG = 3
    wl = S.WORKLOADS[3]
    ppr = 2
    lo = rank * ppr
    mus_h, nus_h = S.batch(3, lo, lo + ppr)
    Nf = mus_h.shape[1]
    args = argparse.Namespace(e2e_steps=2)
    out = bench.run_e2e(args, torch, dist, G, S, wl, "fp32", list(wl.combos), wl.dims, Nf, ppr,
                        rank, world, mus_h, nus_h)
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


def test_bench_e2e_distributed_leg_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_e2e_worker, args=(r, world, port, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        assert got[r]["gather_matches_single_process"] is True
        assert got[r]["gathered_pairs"] == 4
        assert got[r]["value"] > 0 and got[r]["steps"] == 2
    assert got[0]["s_per_step"] == got[1]["s_per_step"]  # max over ranks
