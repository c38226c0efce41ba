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

`--impl reference` times the CPU oracle (oracle/port.py, a restatement of
the reference package, with its C simplex) on all host cores.
"""

from __future__ import annotations

import argparse
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
    """One pair, all four combos, all four bounds -- the reference's own algorithm."""
    cfg, pair, combos = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
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


def cpu_oracle_sample(cfg, n_pairs, workers, first_pair=0):
    """Wall time of n_pairs oracle pairs on `workers` processes."""
    from paper_2506_00976_b200 import synthetic as S

    combos = S.WORKLOADS[cfg].combos
    ctx = _pool_ctx()
    with ctx.Pool(workers) as pool:
        t0 = time.perf_counter()
        per = pool.map(_oracle_pair, [(cfg, first_pair + i, combos) for i in range(n_pairs)],
                       chunksize=1)
        wall = time.perf_counter() - t0
    return wall, per


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------


def run_reference(args):
    rank, world, _ = _env_rank()
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    # W warm-up steps on one small pair per worker (import + first-touch), then
    # K steps, each one pair per core through all four combos of config 3
    ctx = _pool_ctx()
    with ctx.Pool(cores) as pool:
        for _ in range(args.warmup):
            pool.map(_oracle_pair, [(1, 0, ((4, 2.0),))] * cores, chunksize=1)
        times = []
        for s in range(args.steps):
            t0 = time.perf_counter()
            pool.map(_oracle_pair, [(CFG, 1000 + s * cores + i,
                                     ((4, 1.0), (4, 2.0), (8, 1.0), (8, 2.0)))
                                    for i in range(cores)], chunksize=1)
            times.append(time.perf_counter() - t0)
    ms = 1000.0 * statistics.mean(times)
    value = cores / (ms / 1000.0)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg3: 128x128 smooth random fields, kappa{4,8} x p{1,2}, "
                               "4 quantization bounds", "pairs_per_step": cores,
                   "parallelism": f"{cores} host processes"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{cores} cfg3 pairs per step (one per core), all 4 combos"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------


def run_b200(args):
    import torch
    import torch.distributed as dist

    rank, world, local = _env_rank()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2506_00976_b200 as G
    from paper_2506_00976_b200 import _native as N
    from paper_2506_00976_b200 import engine as E
    from paper_2506_00976_b200 import synthetic as S
    from paper_2506_00976_b200.device import stream, to_dev

    global CFG
    CFG = args.config
    wl = S.WORKLOADS[CFG]
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
        bt = E.make_batch(mus, nus, dims, k, p, wl.precision)
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

    def step(events, concurrent=len(stages) > 1):  # one combination: nothing to overlap
        nonlocal launches_per_step
        launches = 0
        base = torch.cuda.current_stream()  # the capture stream under graph capture
        events[-1][0].record(base)  # step start
        for ci, (k, p, bt, dp) in enumerate(stages):
            ev = events[ci]
            if not concurrent:  # stage timing pass: everything on one stream
                launches += combo(ci, k, p, bt, dp, ev, base)
                continue
            sc = streams[ci]
            sc.wait_stream(base)
            with torch.cuda.stream(sc):
                launches += combo(ci, k, p, bt, dp, ev, sc)
        for sc in streams if concurrent else ():
            base.wait_stream(sc)
        events[-1][1].record(base)  # step end
        launches_per_step = launches

    class _NoEvent:
        def record(self, stream=None):
            pass

    no_events = [[_NoEvent()] * 7 for _ in stages] + [[_NoEvent()] * 2]

    def combo(ci, k, p, bt, dp, ev, sc):
        launches = 0
        if True:
            ev[0].record(sc)
            bt.pool()
            launches += 2 + (0 if bt.pdims == bt.dims else 2)
            ev[1].record(sc)
            E._cbar(bt)
            # moments x2 + C-bar (p = 2); fp32 diag C-bar: nu pad, 2 reciprocals + C-bar
            launches += 3 if bt.p == 2.0 else (4 if bt.mode == 1 else 1)
            ev[2].record(sc)
            E.launch_primal(bt, dp, wl.max_iter)
            # ipf_fast + TV/moments + pricing + finish (fp32 mode); the exact
            # path adds two arc-coordinate packs and the block map
            launches += (4 if bt.mode == 1 else 7) + (0 if bt.p == 2.0 else 1)  # + arc rows
            ev[3].record(sc)
            E.launch_dual_prep(bt, dp)
            launches += 2
            ev[4].record(sc)
            E.launch_ctransform(bt, dp, 0)
            ev[5].record(sc)
            E.launch_ctransform(bt, dp, 1)
            ev[6].record(sc)
            # separable passes + dot (p = 2); fp32 pruned: cost table, tile max,
            # pruned kernel, dot, plus one f64->f32 conversion of f_hat
            per_ct = (bt.d + 1) if bt.p == 2.0 else (4 if dp.dt == 1 else 2)
            launches += 2 * per_ct + (1 if bt.p != 2.0 and dp.dt == 1 else 0)
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
    serial_ms = statistics.mean(ev[-1][0].elapsed_time(ev[-1][1]) for ev in serial_events)
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
    stage_ms = {}  # (combo, stage) -> mean ms
    for ci, (k, p, _, _) in enumerate(stages):
        for si, nm in enumerate(names):
            stage_ms[(k, p, nm)] = statistics.mean(
                ev[ci][si].elapsed_time(ev[ci][si + 1]) for ev in serial_events)
    ms = statistics.mean(step_ms)
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = ppr * world / (ms / 1000.0)

    # ---- roofline of the dominant kernel --------------------------------
    sink = torch.empty(1, dtype=torch.float32, device="cuda")
    iters = 4096
    blocks = 148 * 8
    N.check(N.lib().gdt_probe_fp32(blocks, 64, N.ptr(sink), stream()), "probe")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cur)
    N.check(N.lib().gdt_probe_fp32(blocks, iters, N.ptr(sink), stream()), "probe")
    e1.record(cur)
    torch.cuda.synchronize()
    fp32_probe = 2.0 * blocks * 256 * 8 * iters / (e0.elapsed_time(e1) / 1000.0) / 1e12
    # denominator: the nominal FP32 CUDA-core rate at the SM clock sampled under
    # load (SMs x 128 FMA lanes x 2 FLOP x f); the FFMA probe is reported beside it
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    fp32_peak = sms * 128 * 2.0 * float(clk.get("sm_mhz") or 1965.0) * 1e6 / 1e12
    peak_src = (f"nominal {sms} SMs x 128 FP32 lanes x 2 at the sampled {clk.get('sm_mhz')} MHz; "
                f"FFMA probe measured {fp32_probe:.1f} TFLOP/s")
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
    # algorithmic bytes: 48 B per cell and executed sweep
    # (read b, mu, write a; read a, nu, write b) + 32 B per cell for TV and
    # pricing.  ipf_fast_kernel (fp32 mode) moves fewer: it recomputes a and
    # b from mu, nu and the per-block denominators instead of storing them
    # every sweep (16 B per cell and sweep; the ncu DRAM traffic is in profiles/).
    ipf_bytes = (48.0 * sweeps + 32.0) * Nf * ppr
    bytes_model = "(48*S + 32) * N^d bytes per pair (SURVEY.md 8(d))"
    ipf_roof = {"bound": "hbm", "kernel": ("ipf_fast_kernel" if wl.precision == "fp32" else
                                           "ipf_kernel") + " + moments_tv + price (primal stage)",
                "achieved": ipf_bytes / (prim_ms / 1000.0) / 1e9, "peak": hbm, "unit": "GB/s",
                "frac": ipf_bytes / (prim_ms / 1000.0) / 1e9 / hbm,
                "traffic": traffic("ipf_fast_kernel") if wl.precision == "fp32" else None,
                "traffic_source": tsrc, "sweeps": sweeps,
                "work": bytes_model + "; stage time includes pricing"}

    ct_roofs = {}
    for (k, p_, nm), v in stage_ms.items():
        if nm in ("ct_target", "ct_source") and p_ != 2.0:
            eff = 2.0 * Nf * Nf * ppr / (v / 1000.0) / 1e12
            ct_roofs[f"k{k}_p{p_:g}_{nm}"] = round(eff, 3)
    ct_roof = None
    if ct_roofs:
        best = max(ct_roofs.values())
        ct_roof = {"bound": "fp32", "kernel": "pruned_ct_kernel (fp32, p != 2)",
                   "achieved": best, "peak": fp32_peak, "unit": "TFLOP/s",
                   "frac": best / fp32_peak, "traffic": traffic("pruned_ct_tab_kernel"),
                   "traffic_source": tsrc, "per_launch": ct_roofs,
                   "peak_source": peak_src,
                   "work": "brute-force count 2*N^4 per transform per pair (the reference's "
                           "algorithm); tile pruning evaluates a subset exactly, so this is an "
                           "effective rate"}
    if rl is None:
        rl = dict(ipf_roof) if dname == "primal" else {"bound": "hbm", "kernel": dname,
                                                         "achieved": None, "peak": hbm,
                                                         "unit": "GB/s", "frac": None,
                                                         "traffic": None}
    line = {
        "metric": METRIC if CFG == 3 else
        f"pairs/sec for the four quantization bounds, BASELINE config {CFG} "
        f"({'x'.join(map(str, dims))}, combos {list(combos)})",
        "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "fp32+f64",
        "data": "synthetic (seeded smooth random fields, BASELINE.json config 3)",
        "config": {"workload": ("cfg3: 45 pairs/GPU of 128x128 smooth random fields; "
                                "kappa in {4,8} x p in {1,2}; 4 quantization bounds; fp32 mode")
                   if CFG == 3 else f"cfg{CFG}: {ppr} pairs/GPU of {wl.kind} on "
                   f"{'x'.join(map(str, dims))}; {wl.precision} mode; max_iter {wl.max_iter}",
                   "pairs_per_gpu": ppr, "global_pairs": ppr * world, "grid": list(dims),
                   "combos": [list(c) for c in combos],
                   "parallelism": f"dp{world} (pairs sharded, no data-path collective)",
                   "l2": "flushed (256 MB write) between timed steps",
                   "lp": "coarse LP plans precomputed on the host (timed in e2e)",
                   "setup_s": t_setup,
                   "streams": ("one CUDA stream per (kappa, p) combination, forked from and "
                               "joined into the timed stream; stage_ms from a serial pass")
                              if len(stages) > 1 else "one stream",
                   "graph": graph_note,
                   "serial_ms_per_step": round(serial_ms, 4),
                   "streams_match_serial": streams_match,
                   "stage_ms": {f"k{k}_p{p:g}_{nm}": round(v, 4)
                                for (k, p, nm), v in sorted(stage_ms.items())}},
        "roofline": rl, "roofline_ipf": ipf_roof, "roofline_ctransform": ct_roof, "clocks": clk,
        "gpu_launches": launches_per_step * args.steps,
    }

    # ---- e2e through the public API with host buffers --------------------
    if not args.no_e2e:
        # each rank gets its own slice of the host cores for its LPs
        lp_threads = max(1, (os.cpu_count() or 1) // world)
        pin_mu = torch.from_numpy(mus_h).pin_memory()
        pin_nu = torch.from_numpy(nus_h).pin_memory()
        h2d = d2h = 0
        # one public-API call per step for all (kappa, p) combinations: the
        # masses go up once and the coarse LPs of every combination share one
        # host thread pool (quantized_bounds_many)
        G.quantized_bounds_many(pin_mu, pin_nu, dims, combos, precision=wl.precision, xi=wl.xi,
                                max_iter=wl.max_iter, lp_threads=lp_threads)  # untimed warm-up
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        parts = {}
        for _ in range(args.e2e_steps):
            tm = {}
            res = G.quantized_bounds_many(pin_mu, pin_nu, dims, combos, precision=wl.precision,
                                          xi=wl.xi, max_iter=wl.max_iter, timings=tm,
                                          lp_threads=lp_threads)
            for key, val in tm.items():
                if isinstance(val, float):
                    parts[key] = parts.get(key, 0.0) + val
            h2d += 2 * ppr * Nf * 8
            for k, p in combos:
                n_c = Nf // k ** len(dims)
                d2h += ppr * (n_c * n_c * 8 + 2 * n_c * 8 + 8 * 8 + 2 * 8)
                reps = res[(k, float(p))]
                assert all(not isinstance(r[m], Exception) for r in reps for m in r)
        torch.cuda.synchronize()
        e2e_s = (time.perf_counter() - t0) / args.e2e_steps
        if world > 1:
            t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        line["e2e"] = {"value": ppr * world / e2e_s, "unit": UNIT,
                       "h2d_bytes_per_step": h2d // args.e2e_steps,
                       "d2h_bytes_per_step": d2h // args.e2e_steps,
                       "s_per_step": e2e_s, "host_cores": os.cpu_count(),
                       "lp_threads_per_rank": lp_threads,
                       "breakdown_s": {k: round(v / args.e2e_steps, 4) for k, v in parts.items()},
                       "note": "public API quantized_bounds_many (all combos, one call per "
                               "step) from pinned host memory; includes 3 host LPs per pair "
                               "per combo on the rank's host cores"}

    # ---- CPU baseline (rank 0, N=1 only) --------------------------------
    if world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        wall, per = cpu_oracle_sample(CFG, cores, cores, first_pair=1000)
        line["cpu_baseline"] = {
            "value": cores / wall, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{cores} cfg3 pairs (one per core, all 4 combos x 4 bounds); "
                      f"{statistics.mean(per):.1f} s per pair per core",
        }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
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
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches, no CUDA graph")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
