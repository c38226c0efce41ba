"""Stream discipline of the C ABI (GPU).

Every entry point takes the caller's stream and launches only on it (no
default-stream kernels, no shared scratch), so independent (kappa, p)
combinations may run concurrently on their own streams -- bench.py does.
Running SumPool, C-bar and the primal / dual device stages of four
combinations on four streams at once must reproduce the one-stream results
bit for bit.
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

G = pytest.importorskip("paper_2506_00976_b200")
import paper_2506_00976_b200.engine as E  # noqa: E402


def _stages(mus, nus, dims):
    out = []
    for kappa in (4, 8):
        for p in (1.0, 2.0):
            bt = E.make_batch(mus, nus, dims, kappa, p, precision="fp32")
            plans = E.prepare_coarse(bt, E.QUANT_METHODS, lp_threads=0)
            out.append((bt, E.DevicePlans(bt, plans, None, None)))
    return out


def _run(bt, dp):
    bt.pool()
    cbar, _ = E._cbar(bt)
    E.gpu_stages(bt, dp, E.QUANT_METHODS, max_iter=2000)
    return cbar


def test_concurrent_streams_match_serial():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    dims = (64, 64)
    rng = np.random.default_rng(7)
    mus, nus = rng.random((5, 4096)), rng.random((5, 4096))
    mus /= mus.sum(1, keepdims=True)
    nus /= nus.sum(1, keepdims=True)
    stages = _stages(mus, nus, dims)

    serial = []
    for bt, dp in stages:
        cbar = _run(bt, dp)
        serial.append((cbar.clone(), dp.prim_out.clone(), dp.dots.clone(), dp.ff.clone()))
    torch.cuda.synchronize()

    cur = torch.cuda.current_stream()
    streams = [torch.cuda.Stream() for _ in stages]
    for rep in range(3):
        for (bt, dp) in stages:  # clobber the outputs before the concurrent run
            dp.prim_out.fill_(float("nan"))
            dp.dots.fill_(float("nan"))
            dp.ff.fill_(float("nan"))
        conc = []
        for (bt, dp), s in zip(stages, streams):
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                conc.append(_run(bt, dp))
        for s in streams:
            cur.wait_stream(s)
        torch.cuda.synchronize()
        for (cb, po, dots, ff), c, (bt, dp) in zip(serial, conc, stages):
            assert torch.equal(c, cb), (bt.kappa, bt.p, rep)
            assert torch.equal(dp.prim_out, po), (bt.kappa, bt.p, rep)
            assert torch.equal(dp.dots, dots), (bt.kappa, bt.p, rep)
            assert torch.equal(dp.ff, ff), (bt.kappa, bt.p, rep)
