#!/usr/bin/env python
"""Benchmark: certified W_p bounds for 128x128 image pairs (BASELINE.json config 3).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P bench.py --gpus N ...

A STEP = one batch of 45 seeded synthetic 128x128 pairs per GPU, each pair
evaluated at all four (kappa, p) in {4, 8} x {1, 2} and all four quantization
bounds (weighted-cost UB, primal-upscaling UB, min-cost LB, dual-upscaling
LB), fp32 mode.  `value` = pairs/s over all ranks (weak scaling: 45 pairs per
GPU) for the DEVICE stages with inputs resident in HBM and the coarse LP
plans precomputed (the LP stays on the host by design and is timed in
`e2e`).  `e2e` = the same pairs through the public API
(``quantized_bounds``) from pinned host buffers, host LPs included.

`--impl reference` times the stock reference package (gridot's own four bound
functions and numba simplex, staged byte-identical and sha256-verified in
oracle/_ref/ by build()) on all host cores, on the same seeded pairs.
"""

from __future__ import annotations

import argparse
import contextlib
import json
import os
import statistics
import subprocess
import sys
import threading
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402

CFG = 3
METRIC = "image pairs/sec for upper+lower W_p bounds at 128x128 (4 bounds x kappa{4,8} x p{1,2})"
UNIT = "pairs/s"


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------


def _env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=5)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def _oracle_pair(args):
    """One pair, all its combos, all four bounds -- the reference's own algorithm.

    kind "reference": the stock reference package (oracle/_ref/gridot, staged
    byte-identical by build(), sha256-verified, numba simplex); kind "port":
    the oracle's numpy restatement (used only if the staged copy is absent)."""
    cfg, pair, combos, kind = args
    if kind == "reference":
        from oracle import ref_stock

        return ref_stock.pair_bounds(cfg, pair, combos)[0]
    from oracle import port as P
    from paper_2506_00976_b200 import synthetic as S

    wl = S.WORKLOADS[cfg]
    mu, nu = S.measure(cfg, pair, 0), S.measure(cfg, pair, 1)
    t0 = time.perf_counter()
    for k, p in combos:
        P.four_bounds(mu, nu, wl.dims, k, p, xi=wl.xi, max_iter=wl.max_iter)
    return time.perf_counter() - t0


def _pool_ctx():
    import multiprocessing as mp

    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
    return mp.get_context("fork")


def cpu_kind():
    """("reference", note) when the staged stock reference verifies, else ("port", why)."""
    from oracle import ref_stock

    try:
        ref_stock.verify()
    except ref_stock.ReferenceUnavailable as exc:
        return "port", str(exc)
    # JIT the numba simplex once in the parent (fork inherits it), untimed
    return "reference", f"stock gridot (sha256-pinned copy), numba warm-up {ref_stock.warm_up():.1f} s"


def cpu_sample(cfg, pairs, workers, kind):
    """Wall time of the given pairs (all combos each) on `workers` processes."""
    from paper_2506_00976_b200 import synthetic as S

    combos = S.WORKLOADS[cfg].combos
    ctx = _pool_ctx()
    with ctx.Pool(workers) as pool:
        t0 = time.perf_counter()
        per = pool.map(_oracle_pair, [(cfg, i, combos, kind) for i in pairs], chunksize=1)
        wall = time.perf_counter() - t0
    return wall, per


def measure_peaks(torch, N, stream, cur):
    """FP32 / FP64 CUDA-core peaks measured live (csrc/probes.cu): 148 x 8
    CTAs of 8 independent FMA chains per thread; best of 3 launches each."""
    sink = torch.empty(1, dtype=torch.float32, device="cuda")
    blocks, out = 148 * 8, {}
    for name, kind, iters in (("ffma", 0, 256), ("ffma2", 1, 128), ("dfma", 2, 256)):
        N.check(N.lib().gdt_probe_peak(kind, blocks, 8, N.ptr(sink), stream()), "probe")
        best = None
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(cur)
            N.check(N.lib().gdt_probe_peak(kind, blocks, iters, N.ptr(sink), stream()), "probe")
            e1.record(cur)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        out[f"{name}_tflops"] = N.lib().gdt_probe_flops(kind, blocks, iters) / (best / 1e3) / 1e12
    out["fp32_tflops"] = max(out["ffma_tflops"], out["ffma2_tflops"])
    out["fp64_tflops"] = out["dfma_tflops"]
    # dependent-DADD latency: what one add of an exact-order IPF chain costs
    cyc = torch.zeros(1, dtype=torch.int64, device="cuda")
    for _ in range(2):
        N.check(N.lib().gdt_probe_dadd_chain(8192, N.ptr(cyc), stream()), "probe")
        torch.cuda.synchronize()
    out["dadd_chain_cycles_per_add"] = float(cyc[0]) / 8192.0
    return out


def _ref_pairs(step, cores, total):
    """Pairs of CPU step `step`: the GPU arm's own seeds (pairs 0..total-1), in turn."""
    return [(step * cores + i) % total for i in range(cores)]


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------


def run_reference(args):
    rank, world, _ = _env_rank()
    if rank != 0:
        return 0
    from paper_2506_00976_b200 import synthetic as S

    cfg = args.config
    wl = S.WORKLOADS[cfg]
    total = args.pairs or (45 if cfg == 4 else wl.pairs)
    cores = os.cpu_count() or 1
    kind, note = cpu_kind()
    ctx = _pool_ctx()
    # W warm-up steps (one small config-1 pair per worker: imports, first
    # touch, numba cache load), then K steps of one benched pair per core
    # through every (kappa, p) combination and all four bounds
    with ctx.Pool(cores) as pool:
        for _ in range(args.warmup):
            pool.map(_oracle_pair, [(1, 0, ((4, 2.0),), kind)] * cores, chunksize=1)
        times, per = [], []
        for s in range(args.steps):
            t0 = time.perf_counter()
            per += pool.map(_oracle_pair, [(cfg, i, wl.combos, kind)
                                           for i in _ref_pairs(s, cores, total)], chunksize=1)
            times.append(time.perf_counter() - t0)
    ms = 1000.0 * statistics.mean(times)
    value = cores / (ms / 1000.0)
    sample = (f"{cores} cfg{cfg} pairs per step (one per core; seeds = the GPU arm's pairs "
              f"0..{total - 1}), all {len(wl.combos)} (kappa, p) x 4 bounds; "
              f"{statistics.mean(per):.1f} s per pair per core")
    line = {
        "impl": "reference", "metric": _metric(cfg, wl), "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": _workload(cfg, wl, total), "pairs_per_step": cores,
                   "parallelism": f"{cores} host processes", "same_config": True},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": sample, "source": note},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _metric(cfg, wl):
    if cfg == 3:
        return METRIC
    return (f"pairs/sec for the four quantization bounds, BASELINE config {cfg} "
            f"({'x'.join(map(str, wl.dims))}, combos {list(wl.combos)})")


def _workload(cfg, wl, ppr):
    if cfg == 3:
        return ("cfg3: 45 pairs/GPU of 128x128 smooth random fields; kappa in {4,8} x p in "
                "{1,2}; 4 quantization bounds; " + wl.precision + " mode")
    return (f"cfg{cfg}: {ppr} pairs/GPU of {wl.kind} on {'x'.join(map(str, wl.dims))}; "
            f"{wl.precision} mode; max_iter {wl.max_iter}")


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------


def run_e2e(args, torch, dist, G, S, wl, prec, combos, dims, Nf, ppr, rank, world, mus_h, nus_h):
    """The same job through the public API, from pinned host buffers, host LPs
    included.  One call per step for all (kappa, p) combinations
    (quantized_bounds_many: masses uploaded once, every combination's coarse
    LPs on one host thread pool).  Under torchrun the job is the global batch
    of ppr * world pairs through distributed_bounds_many: each rank computes
    its contiguous shard, and one NCCL all_gather collects the per-pair
    bound records on every rank.  Each rank gets cores // world host threads
    for its LPs, so the host's LP capacity is the e2e ceiling at any N."""
    from paper_2506_00976_b200 import distributed as D

    cuda = torch.cuda.is_available()  # (the CPU test of this path runs it under gloo)
    dev = torch.device("cuda", torch.cuda.current_device()) if cuda else torch.device("cpu")
    sync = torch.cuda.synchronize if cuda else (lambda: None)
    pin = (lambda t: t.pin_memory()) if cuda else (lambda t: t)
    lp_threads = max(1, (os.cpu_count() or 1) // world)
    total = ppr * world
    lo, hi = rank * ppr, (rank + 1) * ppr
    if world > 1:
        # global host arrays; this rank fills (and reads) its own shard only
        g_mu = pin(torch.zeros((total, Nf), dtype=torch.float64))
        g_nu = pin(torch.zeros((total, Nf), dtype=torch.float64))
        g_mu[lo:hi] = torch.from_numpy(mus_h)
        g_nu[lo:hi] = torch.from_numpy(nus_h)
        assert D.shard_range(total, rank, world) == (lo, hi)
    else:
        g_mu = pin(torch.from_numpy(mus_h))
        g_nu = pin(torch.from_numpy(nus_h))
    kw = dict(precision=prec, xi=wl.xi, max_iter=wl.max_iter, lp_threads=lp_threads)

    def call(timings=None):
        if world > 1:
            return D.distributed_bounds_many(g_mu, g_nu, dims, combos, timings=timings, **kw)
        res = G.quantized_bounds_many(g_mu, g_nu, dims, combos, timings=timings, **kw)
        return res, None

    call()  # untimed warm-up
    sync()
    if world > 1:
        dist.barrier()
    times, parts, table = [], {}, None
    for _ in range(args.e2e_steps):
        tm = {}
        t0 = time.perf_counter()
        res, table = call(tm)
        sync()
        times.append(time.perf_counter() - t0)
        for key, val in tm.items():
            if isinstance(val, float):
                parts[key] = parts.get(key, 0.0) + val
    if world == 1:
        for key in res:
            assert all(not isinstance(r[m], Exception) for r in res[key] for m in r)
    e2e_s = statistics.mean(times)
    if world > 1:
        t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    h2d = 2 * ppr * Nf * 8
    d2h = sum(ppr * ((Nf // k ** len(dims)) ** 2 * 8 + 2 * (Nf // k ** len(dims)) * 8 + 80)
              for k, _ in combos)
    out = {"value": total / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "bytes_note": "per rank (its shard's masses up; C-bar, "
           "coarse masses and per-pair results down)",
           "s_per_step": e2e_s, "steps": args.e2e_steps,
           "s_per_step_stats": {"mean": statistics.mean(times), "min": min(times),
                                "max": max(times),
                                "stdev": statistics.stdev(times) if len(times) > 1 else 0.0},
           "host_cores": os.cpu_count(), "lp_threads_per_rank": lp_threads,
           "breakdown_s": {k: round(v / args.e2e_steps, 4) for k, v in parts.items()},
           "note": ("distributed_bounds_many: contiguous pair shards, one NCCL all_gather of "
                    "per-pair records" if world > 1 else "public API quantized_bounds_many") +
                   " (all combos, one call per step) from pinned host memory; includes 3 host "
                   "LPs per pair per combo on the rank's host cores"}
    if world > 1:
        # the gathered table must equal the table of ONE process computing the
        # whole global batch (rank 0, all host cores, untimed), bit for bit
        ok = torch.zeros(1, device=dev)
        if rank == 0:
            a_mu, a_nu = S.batch(CFG, 0, total)
            whole = G.quantized_bounds_many(a_mu, a_nu, dims, combos, precision=prec, xi=wl.xi,
                                            max_iter=wl.max_iter)
            ref = np.stack([D.pack_records(whole[(int(k), float(p))], 0) for k, p in combos])
            same = np.array_equal(np.delete(ref, D._IDX["wall_time"], axis=2),
                                  np.delete(table, D._IDX["wall_time"], axis=2), equal_nan=True)
            ok[0] = 1.0 if same else 0.0
        dist.broadcast(ok, 0)
        out["gather_matches_single_process"] = bool(ok.item() == 1.0)
        out["gathered_pairs"] = int(table.shape[1])
    return out


def run_b200(args):
    import torch
    import torch.distributed as dist

    rank, world, local = _env_rank()
    torch.cuda.set_device(local)
    if world > 1:
        # communicator init lines (rank count, transport) on stderr for the record
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2506_00976_b200 as G
    from paper_2506_00976_b200 import _native as N
    from paper_2506_00976_b200 import engine as E
    from paper_2506_00976_b200 import synthetic as S
    from paper_2506_00976_b200.device import stream, to_dev

    global CFG
    CFG = args.config
    wl = S.WORKLOADS[CFG]
    prec = args.precision or wl.precision
    ppr = args.pairs or (45 if CFG == 4 else wl.pairs)  # cfg4: 360 pairs = 45 per GPU x 8
    lo = rank * ppr
    mus_h, nus_h = S.batch(CFG, lo, lo + ppr)
    dims = wl.dims
    Nf = int(np.prod(dims))
    mus = to_dev(mus_h)
    nus = to_dev(nus_h)
    combos = wl.combos

    # ---- setup (untimed): coarse LP plans for the device-stage benchmark
    stages = []
    t_setup = time.perf_counter()
    for k, p in combos:
        bt = E.make_batch(mus, nus, dims, k, p, prec)
        plans = E.prepare_coarse(bt, E.QUANT_METHODS, lp_threads=0)
        dp = E.DevicePlans(bt, plans, None, wl.xi)
        stages.append((k, p, bt, dp))
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t_setup

    cur = torch.cuda.current_stream()
    names = ("pool", "cbar", "primal", "dual_prep", "ct_target", "ct_source")
    launches_per_step = 0

    # the (kappa, p) combinations are independent: each runs on its own
    # stream, forked from and joined back into the current one, so the
    # latency-bound small kernels of one overlap the big ones of another
    streams = [torch.cuda.Stream() for _ in stages]
    # C-bar of a coarser level is pooled from a finer level's (same p, fp32
    # mode, nested blocks: engine.cbar_parent), as quantized_bounds_many does:
    # that combination's stream waits for its parent's C-bar
    parents = []
    for ci, (_, _, bt, _) in enumerate(stages):
        par = E.cbar_parent(bt, [st_[2] for st_ in stages[:ci]], computed=False)
        parents.append(None if par is None else
                       next(j for j, st_ in enumerate(stages) if st_[2] is par))
    cbar_done = [torch.cuda.Event() for _ in stages]
    # inside a combination the dual chain (f_ext, interpolation, the two
    # c-transforms) needs only the plans and the masses, not C-bar or the
    # primal stage: it runs on a second stream of the combination, forked
    # after the SumPool (at cfg4 the 45-CTA IPF kernel then overlaps the
    # c-transforms instead of idling 100 SMs)
    # Measured: cfg4 1.79 -> 1.59 ms, cfg5 0.685 -> 0.553 ms; with four
    # combinations already on four streams the extra streams only add
    # contention (cfg3 2.22 -> 2.27 ms), so the split is used for
    # single-combination configs.  (fp64 mode, C-bar moved to the dual stream
    # too -- the primal stage does not price with it there: cfg5 0.553 -> 0.567
    # ms, not kept.)
    split_dual = len(stages) == 1
    dual_streams = [torch.cuda.Stream() if split_dual else None for _ in stages]
    pool_done = [torch.cuda.Event() for _ in stages]

    base_stream = [None]

    def step(events, concurrent=True):
        nonlocal launches_per_step
        launches = 0
        base = torch.cuda.current_stream()  # the capture stream under graph capture
        base_stream[0] = base
        events[-1][0].record(base)  # step start
        for ci, (k, p, bt, dp) in enumerate(stages):
            ev = events[ci]
            if not concurrent:  # stage timing pass: everything on one stream
                launches += combo(ci, k, p, bt, dp, ev, base, None)
                continue
            sc = streams[ci]
            sc.wait_stream(base)
            with torch.cuda.stream(sc):
                launches += combo(ci, k, p, bt, dp, ev, sc, dual_streams[ci])
        for sc in (streams + [x for x in dual_streams if x is not None]) if concurrent else ():
            base.wait_stream(sc)
        events[-1][1].record(base)  # step end
        launches_per_step = launches

    class _NoEvent:
        def record(self, stream=None):
            pass

    no_events = [[_NoEvent()] * 7 for _ in stages] + [[_NoEvent()] * 2]

    def combo(ci, k, p, bt, dp, ev, sc, sd):
        launches = 0
        ev[0].record(sc)
        bt.pool()
        launches += 2 + (0 if bt.pdims == bt.dims else 2)
        ev[1].record(sc)
        if sd is not None:
            pool_done[ci].record(sc)

        def upper():  # C-bar, then the primal stage (fp32 mode prices with C-bar)
            n_l = 0
            if parents[ci] is not None:
                sc.wait_event(cbar_done[parents[ci]])
                E._cbar(bt, stages[parents[ci]][2])
                n_l += 1  # the pooling kernel
            else:
                E._cbar(bt)
                # moments x2 + C-bar (p = 2); fp32 diag C-bar: nu pad, 2 reciprocals + C-bar
                n_l += 3 if bt.p == 2.0 else (4 if bt.mode == 1 else 1)
            cbar_done[ci].record(sc)
            ev[2].record(sc)
            E.launch_primal(bt, dp, wl.max_iter)
            # ipf_fast + TV/moments + pricing + finish (fp32 mode); the exact
            # path adds two arc-coordinate packs and the block map
            n_l += (4 if bt.mode == 1 else 7) + (0 if bt.p == 2.0 else 1)  # + arc rows
            ev[3].record(sc)
            return n_l

        def lower():  # the dual chain: needs the plans and the masses only
            n_l = 0
            if sd is not None:
                sd.wait_event(pool_done[ci])
            with (torch.cuda.stream(sd) if sd is not None else contextlib.nullcontext()):
                sx = sd if sd is not None else sc
                E.launch_dual_prep(bt, dp)
                n_l += 2
                ev[4].record(sx)
                E.launch_ctransform(bt, dp, 0)
                ev[5].record(sx)
                E.launch_ctransform(bt, dp, 1)
                ev[6].record(sx)
            # separable passes + dot (p = 2); fp32 pruned: cost table, tile max,
            # pruned kernel, dot, plus one f64->f32 conversion of f_hat
            per_ct = (bt.d + 1) if bt.p == 2.0 else (4 if dp.dt == 1 else 2)
            return n_l + 2 * per_ct + (1 if bt.p != 2.0 and dp.dt == 1 else 0)

        # a combination whose C-bar is pooled from another one's runs its dual
        # chain first instead of waiting for the parent's C-bar (concurrent
        # schedule only: the serial stage-timing pass keeps the stage order)
        if parents[ci] is not None and sc is not base_stream[0]:
            launches += lower() + upper()
        else:
            launches += upper() + lower()
        return launches

    def new_events():
        # per combo: 7 stage boundaries on its stream; last entry: step start / end
        return [[torch.cuda.Event(enable_timing=True) for _ in range(7)] for _ in stages] + \
            [[torch.cuda.Event(enable_timing=True) for _ in range(2)]]

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    for _ in range(args.warmup):
        step(new_events())
    torch.cuda.synchronize()

    # the whole step (all combinations, fork and join included) as one CUDA
    # graph: replays the same launches on the same buffers without the
    # per-launch host cost (ctypes argument marshalling + cudaLaunchKernel)
    graph, graph_note = None, "off (--no-graph)"
    if not args.no_graph:
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                step(no_events)
            g.replay()
            torch.cuda.synchronize()
            graph, graph_note = g, "one CUDA graph per step (captured after warm-up)"
        except Exception as exc:  # capture unsupported: time the eager launches
            graph_note = f"capture failed, eager launches ({type(exc).__name__}: {exc})"[:200]
            print(f"bench: {graph_note}", file=sys.stderr)
            torch.cuda.synchronize()

    def timed_step(ev):
        if graph is None:
            step(ev)
            return
        ev[-1][0].record(cur)
        graph.replay()
        ev[-1][1].record(cur)

    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    all_events = []
    for _ in range(args.steps):
        flush.zero_()  # L2 flush (> 126 MB) between timed steps, outside the events
        ev = new_events()
        timed_step(ev)
        all_events.append(ev)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()

    # per-kernel stage times come from an untimed serial pass (one stream, the
    # same flushed-L2 steps): under the concurrent schedule a stage's events
    # would include the kernels of the other combinations running beside it
    conc_out = [(dp.prim_out.clone(), dp.dots.clone()) for _, _, _, dp in stages]
    step(new_events(), concurrent=False)  # warm the current stream's allocator pool
    serial_events = []
    for _ in range(args.steps):
        flush.zero_()
        ev = new_events()
        step(ev, concurrent=False)
        serial_events.append(ev)
    torch.cuda.synchronize()
    serial_ms = statistics.median(ev[-1][0].elapsed_time(ev[-1][1]) for ev in serial_events)
    # the concurrent schedule must not change a single bit of the outputs
    streams_match = all(torch.equal(a, dp.prim_out) and torch.equal(b, dp.dots)
                        for (a, b), (_, _, _, dp) in zip(conc_out, stages))

    # kernels of one step, counted exactly by the CUDA activity profiler on an
    # extra (untimed) step; the hand count of step() is the fallback
    try:
        from torch.profiler import ProfilerActivity, profile

        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            step(new_events())
            torch.cuda.synchronize()
        counted = sum(1 for e in prof.events()
                      if e.device_type.name == "CUDA" and "gdt::" in e.name)
        if os.environ.get("GDT_BENCH_LAUNCHES"):
            import collections
            cnt = collections.Counter(e.name for e in prof.events()
                                      if e.device_type.name == "CUDA" and "gdt::" in e.name)
            print(f"launches: hand {launches_per_step} profiler {counted}: {dict(cnt)}",
                  file=sys.stderr)
        if counted > 0:
            launches_per_step = counted
    except Exception as exc:  # profiler unavailable: keep the hand count
        print(f"launch count: profiler unavailable ({exc}); using the hand count",
              file=sys.stderr)
    step_ms = [ev[-1][0].elapsed_time(ev[-1][1]) for ev in all_events]
    # (combo, stage) -> ms: the MEDIAN over the serial steps -- the first
    # kernel after the L2 flush sometimes runs into the flush's write-back
    # (one step of five at 0.9 ms instead of 0.65 ms), which a mean carries
    # into the roofline fractions
    stage_ms = {}
    for ci, (k, p, _, _) in enumerate(stages):
        for si, nm in enumerate(names):
            stage_ms[(k, p, nm)] = statistics.median(
                ev[ci][si].elapsed_time(ev[ci][si + 1]) for ev in serial_events)
    ms = statistics.mean(step_ms)
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = ppr * world / (ms / 1000.0)

    # ---- roofline of the dominant kernel --------------------------------
    probes = measure_peaks(torch, N, stream, cur)
    fp32_peak = probes["fp32_tflops"]
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    nominal = sms * 128 * 2.0 * float(clk.get("sm_mhz") or 1965.0) * 1e6 / 1e12
    peak_src = (f"measured: max of the FFMA ({probes['ffma_tflops']:.1f}) and packed FFMA2 "
                f"({probes['ffma2_tflops']:.1f}) probes (gdt_probe_peak, this run, kernel timed "
                f"alone); nominal {sms} SMs x 128 lanes x 2 at {clk.get('sm_mhz')} MHz = "
                f"{nominal:.1f}")
    dom = max(stage_ms.items(), key=lambda kv: kv[1])
    (dk, dpow, dname), dms = dom
    n_c = Nf // dk ** len(dims)
    if dname in ("ct_target", "ct_source") and dpow != 2.0:
        flops = 2.0 * Nf * Nf * ppr            # sub + min per candidate
        rl = {"bound": "fp32", "kernel": f"pruned_ct_kernel (c-transform, kappa={dk}, p={dpow:g})"}
    elif dname == "cbar" and dpow != 2.0:
        flops = 2.0 * Nf * Nf * ppr            # one FMA per (row cell, column cell)
        rl = {"bound": "fp32", "kernel": f"cbar_diag_kernel (fp32 FFMA2 C-bar, kappa={dk}, p={dpow:g})"}
    else:
        flops = None
        rl = None
    if flops is not None:
        achieved = flops / (dms / 1000.0) / 1e12
        rl.update({"achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
                   "frac": achieved / fp32_peak, "traffic": None,
                   "peak_source": peak_src,
                   "work": "2 FP32 ops x N^4 candidates per pair (N=128)"})
    # DRAM traffic per launch of the named kernels, from the committed ncu
    # full-set capture of this config (scripts/ncu_traffic.py); None if absent
    tfile = os.path.join(HERE, "profiles", f"ncu_traffic_cfg{CFG}.json")
    try:
        traffic_tab = json.load(open(tfile))
    except (OSError, ValueError):
        traffic_tab = {}

    def traffic(prefix):
        vals = [v["bytes_per_launch"] for k, v in traffic_tab.items() if k.startswith(prefix)]
        return sum(vals) / len(vals) if vals else None

    tsrc = f"profiles/ncu_traffic_cfg{CFG}.json (dram read+write per launch, ncu --set full)"
    if rl is not None:
        kname = (f"cbar_diag_kernel<{dk}," if dname == "cbar" else "pruned_ct_tab_kernel")
        rl["traffic"] = traffic(kname)
        rl["traffic_source"] = tsrc
    # IPF/TV kernel against HBM (north-star secondary roofline)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(HERE, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    prim_ms = statistics.mean(stage_ms[(k, p, "primal")] for k, p, _, _ in stages)
    sweeps = statistics.mean(
        float(np.mean(E.to_host(dp.prim_out)[:, 4])) for _, _, _, dp in stages)
    coarse = prec == "fp32" and all(bt.cbar_dev is not None for _, _, bt, _ in stages)
    if coarse:
        # fp32 mode: the sweeps run on the coarse plan in shared memory
        # (O(arcs) per sweep, latency-bound, not a bandwidth stage); the one
        # fine pass is the weighted TV: read mu and nu once, 16 B per cell
        # (the TV weights and block map are per-grid tables shared by the batch)
        ipf_bytes = 16.0 * Nf * ppr
        ipf_roof = {"bound": "hbm",
                    "kernel": "tv_pass_kernel + primal_coarse_kernel (fp32 primal stage)",
                    "work": "16 * N^d bytes per pair (one read of mu, nu by the weighted-TV "
                            "pass); stage time includes the coarse sweeps and the fold"}
    else:
        # fp64 mode, exact order: 48 B per cell and executed
        # sweep (read b, mu, write a; read a, nu, write b) + 32 B per cell for
        # TV and pricing
        ipf_bytes = (48.0 * sweeps + 32.0) * Nf * ppr
        ipf_roof = {"bound": "hbm",
                    "kernel": "ipf_cluster_kernel / ipf_kernel + moments_tv + price (primal stage)",
                    "work": "(48*S + 32) * N^d bytes per pair (SURVEY.md 8(d)); stage time "
                            "includes the run lists and pricing",
                    "note": "the exact-order unit sums are sequential DADD chains "
                            f"({probes['dadd_chain_cycles_per_add']:.1f} cycles per add measured): "
                            "the stage is latency-bound, the HBM fraction is reported as the "
                            "north star asks"}
    ipf_roof.update({"achieved": ipf_bytes / (prim_ms / 1000.0) / 1e9, "peak": hbm,
                     "unit": "GB/s", "frac": ipf_bytes / (prim_ms / 1000.0) / 1e9 / hbm,
                     "traffic": traffic("tv_pass_kernel") if coarse else
                     (traffic("ipf_cluster_kernel") or traffic("ipf_kernel")),
                     "traffic_source": tsrc, "sweeps": sweeps, "stage_ms": round(prim_ms, 4)})

    # the pooled C-bar (nested levels): a pure streaming pass, against HBM
    pool_roof = None
    for ci, pj in enumerate(parents):
        if pj is None:
            continue
        kc, pc, btc, _ = stages[ci]
        btf = stages[pj][2]
        nbytes = 8.0 * ppr * (btf.n * btf.n + btc.n * btc.n + 2 * btf.n + 2 * btc.n) + 8.0 * btc.n ** 2
        t_ms = stage_ms[(kc, pc, "cbar")]
        pool_roof = {"bound": "hbm", "kernel": f"cbar_pool_kernel (C-bar kappa={kc} from kappa={stages[pj][0]}, p={pc:g})",
                     "achieved": nbytes / (t_ms / 1000.0) / 1e9, "peak": hbm, "unit": "GB/s",
                     "frac": nbytes / (t_ms / 1000.0) / 1e9 / hbm,
                     "traffic": traffic("cbar_pool_kernel"), "traffic_source": tsrc,
                     "work": "8 (n_f^2 + n^2) bytes per pair: the finer C-bar read once, the "
                             "coarser one written (plus the coarse masses and centre costs)",
                     "stage_ms": round(t_ms, 4)}
    ct_roofs = {}
    for (k, p_, nm), v in stage_ms.items():
        if nm in ("ct_target", "ct_source") and p_ != 2.0:
            eff = 2.0 * Nf * Nf * ppr / (v / 1000.0) / 1e12
            ct_roofs[f"k{k}_p{p_:g}_{nm}"] = round(eff, 3)
    ct_roof = None
    if ct_roofs:
        best_key = max(ct_roofs, key=ct_roofs.get)
        best = ct_roofs[best_key]
        ct_roof = {"bound": "fp32", "kernel": "pruned_ct_tab_kernel (fp32, p = 1)",
                   "achieved": best, "peak": fp32_peak, "unit": "TFLOP/s",
                   "frac": best / fp32_peak, "traffic": traffic("pruned_ct_tab_kernel"),
                   "traffic_source": tsrc, "per_launch": ct_roofs,
                   "peak_source": peak_src,
                   "work": "brute-force-equivalent count 2*N^4 per transform per pair (the "
                           "reference's algorithm); tile pruning evaluates a subset exactly, so "
                           "achieved/frac are effective rates"}
        # executed-candidate rate: the evaluated fraction of source tiles,
        # counted by the trace build (scripts/ct_trace.py) on this workload
        try:
            tiles = json.load(open(os.path.join(HERE, "profiles", "r02_ct_tiles.json")))
            fr = tiles[best_key.split("_ct")[0]]["evaluated_fraction"]
            ct_roof.update({"evaluated_fraction": fr, "achieved_executed": best * fr,
                            "frac_executed": best * fr / fp32_peak,
                            "executed_source": "profiles/r02_ct_tiles.json (scripts/ct_trace.py, "
                                               "trace build, same 45 cfg3 pairs)"})
        except (OSError, ValueError, KeyError):
            pass
    if rl is None:
        rl = dict(ipf_roof) if dname == "primal" else {"bound": "hbm", "kernel": dname,
                                                         "achieved": None, "peak": hbm,
                                                         "unit": "GB/s", "frac": None,
                                                         "traffic": None}
    line = {
        "metric": _metric(CFG, wl),
        "value": value if streams_match else None, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None,
        "dtype": "fp32+f64" if prec == "fp32" else "f64",
        "data": f"synthetic (seeded {wl.kind}, BASELINE.json config {CFG})",
        "config": {"workload": _workload(CFG, wl, ppr).replace(wl.precision + " mode",
                                                                prec + " mode"),
                   "precision": prec,
                   "pairs_per_gpu": ppr, "global_pairs": ppr * world, "grid": list(dims),
                   "combos": [list(c) for c in combos],
                   "parallelism": f"dp{world} (pairs sharded, no data-path collective)",
                   "l2": "flushed (256 MB write) between timed steps",
                   "lp": "coarse LP plans precomputed on the host (timed in e2e)",
                   "setup_s": t_setup,
                   "streams": (("two CUDA streams (SumPool, C-bar, primal | dual chain, forked after "
                                "the SumPool)" if split_dual else
                                "one CUDA stream per (kappa, p) combination") +
                               ", forked from and joined into the timed stream; stage_ms = median "
                               "over a serial pass"),
                   "graph": graph_note,
                   "cbar_pooled": {f"k{stages[ci][0]}_p{stages[ci][1]:g}":
                                   f"from k{stages[pj][0]}_p{stages[pj][1]:g} (nested blocks: the "
                                   "numerator is additive; gdt_weighted_cost_pool)"
                                   for ci, pj in enumerate(parents) if pj is not None},
                   "serial_ms_per_step": round(serial_ms, 4),
                   "streams_match_serial": streams_match,
                   "stage_ms": {f"k{k}_p{p:g}_{nm}": round(v, 4)
                                for (k, p, nm), v in sorted(stage_ms.items())}},
        "roofline": rl, "roofline_ipf": ipf_roof, "roofline_ctransform": ct_roof,
        "roofline_cbar_pool": pool_roof, "clocks": clk,
        "peaks_measured": {k: round(v, 2) for k, v in probes.items()},
        "gpu_launches": launches_per_step * args.steps,
    }

    # ---- e2e through the public API with host buffers --------------------
    if not args.no_e2e:
        line["e2e"] = run_e2e(args, torch, dist, G, S, wl, prec, combos, dims, Nf, ppr, rank,
                              world, mus_h, nus_h)

    # ---- CPU baseline (rank 0, N=1 only) --------------------------------
    if world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        kind, note = cpu_kind()
        wall, per = cpu_sample(CFG, _ref_pairs(0, cores, ppr), cores, kind)
        line["cpu_baseline"] = {
            "value": cores / wall, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"{cores} cfg{CFG} pairs = the first {cores} benched pairs (one per core, "
                      f"all {len(combos)} combos x 4 bounds); "
                      f"{statistics.mean(per):.1f} s per pair per core",
            "source": note,
        }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    if not streams_match:
        # a broken stream or graph schedule must not publish a headline number
        print("bench: concurrent/graph outputs differ from the serial pass; value withheld",
              file=sys.stderr)
        return 1
    return 0


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--pairs", type=int, default=0, help="pairs per GPU (default: the config's)")
    ap.add_argument("--config", type=int, default=3, choices=(1, 2, 3, 4, 5),
                    help="BASELINE.json config (3 = the headline 128x128 workload)")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--precision", choices=("fp64", "fp32"), default=None,
                    help="override the config's precision mode (cfg3 default: fp32)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches, no CUDA graph")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
