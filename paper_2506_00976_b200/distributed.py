"""Data parallelism over independent pairs.

Pairs are independent: each rank (one process per GPU) takes a contiguous
shard, computes its bounds with no data-path collective, and one
``all_gather`` (NCCL over NVLink/NVSwitch on GPUs, gloo in the CPU tests)
collects fixed-width per-pair records so every rank -- rank 0 in practice --
holds the full result table.  Records are F = 16 float64 per pair.
"""

from __future__ import annotations

import math

import numpy as np

from .engine import QUANT_METHODS, quantized_bounds, quantized_bounds_many
from .reports import BoundReport

__all__ = ["shard_range", "RECORD_FIELDS", "pack_records", "unpack_records", "gather_records",
           "gather_records_rows", "distributed_bounds", "distributed_bounds_many"]

RECORD_FIELDS = (
    "pair", "status", "wc_value", "mc_raw", "pu_value", "pu_transport", "pu_delta_mu",
    "pu_delta_nu", "pu_gap", "pu_iterations", "pu_converged", "du_raw", "du_dual_value",
    "coarse_size", "wall_time", "spare",
)
F = len(RECORD_FIELDS)
_IDX = {k: i for i, k in enumerate(RECORD_FIELDS)}
_STATUS_BITS = {m: 1 << i for i, m in enumerate(QUANT_METHODS)}  # bit set = method failed


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) of `total` pairs for `rank`; sizes differ by <= 1."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def pack_records(reports, first_pair: int) -> np.ndarray:
    """[len(reports), F] float64; failed methods set a status bit and NaN values."""
    out = np.full((len(reports), F), np.nan)
    for i, rep in enumerate(reports):
        row = out[i]
        row[_IDX["pair"]] = first_pair + i
        status = 0
        for m in QUANT_METHODS:
            if m in rep and isinstance(rep[m], Exception):
                status |= _STATUS_BITS[m]
        row[_IDX["status"]] = status
        get = lambda m: rep.get(m) if not isinstance(rep.get(m), Exception) else None  # noqa
        wc, mc, pu, du = (get(m) for m in QUANT_METHODS)
        first = next((r for r in (wc, mc, pu, du) if r is not None), None)
        if first is not None:  # shared by every method of the pair
            row[_IDX["coarse_size"]] = np.nan if first.coarse_size is None else first.coarse_size
            row[_IDX["wall_time"]] = first.wall_time
        if wc is not None:
            row[_IDX["wc_value"]] = wc.value
        if mc is not None:
            row[_IDX["mc_raw"]] = mc.raw_value
        if pu is not None:
            row[_IDX["pu_value"]] = pu.value
            for key in ("transport", "delta_mu", "delta_nu"):
                row[_IDX[f"pu_{key}"]] = pu.components[key]
            row[_IDX["pu_gap"]] = pu.components["marginal_gap"]
            row[_IDX["pu_iterations"]] = pu.iterations
            row[_IDX["pu_converged"]] = pu.components["converged"]
        if du is not None:
            row[_IDX["du_raw"]] = du.raw_value
            row[_IDX["du_dual_value"]] = du.components["dual_value"]
    return out


def unpack_records(rec: np.ndarray) -> list[dict]:
    """Inverse of pack_records (exceptions become None)."""
    out = []
    for row in np.asarray(rec):
        st = int(row[_IDX["status"]])
        n = None if math.isnan(row[_IDX["coarse_size"]]) else int(row[_IDX["coarse_size"]])
        wall = 0.0 if math.isnan(row[_IDX["wall_time"]]) else float(row[_IDX["wall_time"]])
        rep = {}
        ok = lambda m: not st & _STATUS_BITS[m]  # noqa: E731
        if ok("weighted_cost") and not math.isnan(row[_IDX["wc_value"]]):
            v = float(row[_IDX["wc_value"]])
            rep["weighted_cost"] = BoundReport("weighted_cost", v, v, {"transport": v}, wall,
                                               None, n)
        if ok("min_cost") and not math.isnan(row[_IDX["mc_raw"]]):
            r = float(row[_IDX["mc_raw"]])
            rep["min_cost"] = BoundReport("min_cost", max(0.0, r), r, {"transport": r}, wall,
                                          None, n)
        if ok("primal_upscaling") and not math.isnan(row[_IDX["pu_value"]]):
            v = float(row[_IDX["pu_value"]])
            comps = {k: float(row[_IDX[f"pu_{k}"]]) for k in ("transport", "delta_mu",
                                                               "delta_nu")}
            comps["marginal_gap"] = float(row[_IDX["pu_gap"]])
            comps["converged"] = float(row[_IDX["pu_converged"]])
            rep["primal_upscaling"] = BoundReport("primal_upscaling", v, v, comps, wall,
                                                  int(row[_IDX["pu_iterations"]]), n)
        if ok("dual_upscaling") and not math.isnan(row[_IDX["du_raw"]]):
            r = float(row[_IDX["du_raw"]])
            rep["dual_upscaling"] = BoundReport("dual_upscaling", max(0.0, r), r,
                                                {"dual_value": float(row[_IDX["du_dual_value"]])},
                                                wall, None, n)
        out.append({"pair": int(row[_IDX["pair"]]), "status": st, "reports": rep})
    return out


def gather_records(local: np.ndarray, total: int, group=None, device=None) -> np.ndarray:
    """All-gather variable-size shards of [n_r, F] records into [total, F] (pair order).

    Shards are padded to the largest shard so one all_gather_into_tensor (NCCL)
    or all_gather (gloo) suffices."""
    return gather_records_rows(local, total, 1, group, device)


def _gather_device(group):
    import torch
    import torch.distributed as dist

    return torch.device("cuda", torch.cuda.current_device()) \
        if dist.get_backend(group) == "nccl" else None


def distributed_bounds(mus, nus, dims, kappa, p, group=None, *, compute=None, **kw):
    """Shard the pairs over the process group, compute, gather records on every rank.

    ``compute(mus, nus, dims, kappa, p, **kw)`` defaults to
    :func:`quantized_bounds` (the CPU tests substitute a host stand-in)."""
    import torch.distributed as dist

    compute = compute or quantized_bounds
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    total = int(mus.shape[0])
    lo, hi = shard_range(total, rank, world)
    reps = compute(mus[lo:hi], nus[lo:hi], dims, kappa, p, **kw) if hi > lo else []
    local = pack_records(reps, lo)
    return unpack_records(gather_records(local, total, group, _gather_device(group)))


def distributed_bounds_many(mus, nus, dims, combos, group=None, *, compute=None, **kw):
    """:func:`distributed_bounds` for several (kappa, p) combinations: each rank
    runs ONE ``quantized_bounds_many`` call on its contiguous shard (its LPs on
    its own host threads), then one all_gather of [pairs x combos, F] records.

    Returns ({(kappa, p): [unpacked record per pair]}, records [combos, total, F])."""
    import torch.distributed as dist

    compute = compute or quantized_bounds_many
    combos = [(int(k), float(p)) for k, p in combos]
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    total = int(mus.shape[0])
    lo, hi = shard_range(total, rank, world)
    res = compute(mus[lo:hi], nus[lo:hi], dims, combos, **kw) if hi > lo else \
        {key: [] for key in combos}
    # records of pair-major rows, combination-minor: [n_r * C, F], gathered in
    # pair order as (total * C) rows
    C = len(combos)
    local = np.stack([pack_records(res[key], lo) for key in combos], axis=1) \
        if hi > lo else np.zeros((0, C, F))
    flat = gather_records_rows(local.reshape(-1, F), total, C, group, _gather_device(group))
    table = flat.reshape(total, C, F).transpose(1, 0, 2).copy()
    return {key: unpack_records(table[j]) for j, key in enumerate(combos)}, table


def gather_records_rows(local: np.ndarray, total: int, per_pair: int, group=None,
                        device=None) -> np.ndarray:
    """gather_records for shards holding `per_pair` consecutive rows per pair."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    width = -(-total // world) * per_pair
    buf = np.full((width, F), np.nan)
    buf[:local.shape[0]] = local
    t = torch.from_numpy(buf)
    if device is not None:
        t = t.to(device)
    if dist.get_backend(group) == "nccl":
        out = torch.empty((world * width, F), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(out, t, group=group)
        parts = [out[r * width:(r + 1) * width] for r in range(world)]
    else:
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t, group=group)
    rows = []
    for r, part in enumerate(parts):
        lo, hi = shard_range(total, r, world)
        rows.append(part[:(hi - lo) * per_pair].cpu().numpy())
    return np.concatenate(rows, axis=0)
