"""The data-parallel path on a real GPU: NCCL process group, world size 1.

Every GPU test runs on one B200, so the NCCL collective is exercised at world
size 1 (the gather path and the record layout are the same at any size; the
multi-rank logic is covered by the gloo world-size-2 tests in
tests/test_distributed.py).  The gathered table must equal the single-process
results bit for bit (wall times aside).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

G = pytest.importorskip("paper_2506_00976_b200")
from paper_2506_00976_b200 import distributed as D  # noqa: E402
from paper_2506_00976_b200 import synthetic as S  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def nccl_group():
    import torch
    import torch.distributed as dist

    if dist.is_initialized():
        yield dist.group.WORLD
        return
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1,
                            device_id=torch.device("cuda", torch.cuda.current_device()))
    yield dist.group.WORLD
    dist.destroy_process_group()


def _strip_wall(table):
    return np.delete(table, D.RECORD_FIELDS.index("wall_time"), axis=-1)


def test_nccl_distributed_bounds_many_equals_single_process(nccl_group):
    import torch.distributed as dist

    assert dist.get_backend(nccl_group) == "nccl"
    wl = S.WORKLOADS[3]
    mus, nus = S.batch(3, 0, 6)
    combos = [(int(k), float(p)) for k, p in wl.combos]
    res, table = D.distributed_bounds_many(mus, nus, wl.dims, combos, precision="fp32",
                                           xi=wl.xi, max_iter=wl.max_iter)
    single = G.quantized_bounds_many(mus, nus, wl.dims, combos, precision="fp32", xi=wl.xi,
                                     max_iter=wl.max_iter)
    want = np.stack([D.pack_records(single[key], 0) for key in combos])
    assert table.shape == (len(combos), 6, D.F)
    assert np.array_equal(_strip_wall(table), _strip_wall(want), equal_nan=True)
    for j, key in enumerate(combos):
        for b in range(6):
            rec = res[key][b]
            assert rec["pair"] == b and rec["status"] == 0
            for m in G.QUANT_METHODS:
                assert rec["reports"][m].raw_value == single[key][b][m].raw_value


def test_nccl_distributed_bounds_single_combo(nccl_group):
    wl = S.WORKLOADS[5]
    mus, nus = S.batch(5, 0, 4)
    recs = D.distributed_bounds(mus, nus, wl.dims, 4, 2.0, precision="fp64", xi=wl.xi)
    single = G.quantized_bounds(mus, nus, wl.dims, 4, 2.0, precision="fp64", xi=wl.xi)
    for b, rec in enumerate(recs):
        for m in G.QUANT_METHODS:
            assert rec["reports"][m].raw_value == single[b][m].raw_value
            assert rec["reports"][m].coarse_size == single[b][m].coarse_size
