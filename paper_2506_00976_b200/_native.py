"""ctypes binding of libgridot_b200.so (include/gridot_b200.h).

The shared library is built in-tree by ``paper_2506_00976_b200.csrc.build``
(``__graft_entry__.build()``).  There is no fallback: if the library is
missing or a CUDA device is required and absent, the calls raise.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import GridotError

_HERE = os.path.dirname(os.path.abspath(__file__))
# GRIDOT_B200_LIB selects another build of the same library (debug / trace
# builds from scripts/); the default is the in-tree release build
LIB_PATH = os.environ.get("GRIDOT_B200_LIB") or os.path.join(_HERE, "csrc", "libgridot_b200.so")

P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int
D = ctypes.c_double

# name -> (restype, argtypes); mirrors include/gridot_b200.h
_SIGNATURES = {
    "gdt_version": (ctypes.c_char_p, []),
    "gdt_last_error": (ctypes.c_char_p, []),
    "gdt_pad_f64": (I32, [P, P, I64, I32, P, I32, P]),
    "gdt_sumpool_f64": (I32, [P, P, I64, I32, P, I32, P]),
    "gdt_sumpool_stats_f64": (I32, [P, P, P, I64, I32, P, I32, P]),
    "gdt_weighted_cost": (I32, [P, P, P, P, P, P, I64, P, P, I64, I32, P, I32, D, I32, P]),
    "gdt_weighted_cost_pool": (I32, [P, P, P, P, P, P, P, P, I64, I32, P, I32, P]),
    "gdt_primal_scratch_bytes": (I64, [I64, I32, P, I32, I32]),
    "gdt_primal_upscale": (I32, [P, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P, I32, P, I64, D,
                                 I64, I32, P, I32, P, I64, I32, P, P, P, P]),
    "gdt_ipf_csr": (I32, [P, P, P, P, P, P, P, P, I64, I64, D, I64, P, P, P, P, P, P, P]),
    "gdt_price_coo": (I32, [P, P, P, I64, P, P, P, I64, D, I32, P, P, P]),
    "gdt_weighted_tv_inner": (I32, [P, P, I64, I32, P, D, P, P, P]),
    "gdt_coarse_ctransform": (I32, [P, P, P, P, I64, I64, P, P]),
    "gdt_interpolate": (I32, [P, P, I64, I32, P, P, P, I32, P]),
    "gdt_ctransform_grid": (I32, [P, P, I64, I32, P, D, I32, I32, P, I64, P, P, P, I64, P]),
    "gdt_ctransform_scratch_bytes": (I64, [I64, I32, P, D, I32]),
    "gdt_ctransform_points": (I32, [P, P, I64, I64, I32, D, P, I32, P, P]),
    "gdt_batched_dot": (I32, [P, P, I64, I64, P, P]),
    "gdt_probe_fp32": (I32, [I64, I64, P, P]),
    "gdt_probe_dadd_chain": (I32, [I64, P, P]),
    "gdt_probe_peak": (I32, [I32, I64, I64, P, P]),
    "gdt_probe_flops": (I64, [I32, I64, I64]),
    "gdt_entropic_scratch_bytes": (I64, [I64, I64]),
    "gdt_entropic_fit": (I32, [P, P, I64, I64, I32, D, D, P, P, D, I64, P, P, P, P, P, P]),
    "gdt_entropic_plan": (I32, [P, P, I64, I64, I32, D, D, P, P, P, P, P, P, P]),
    "gdt_transport_simplex": (I32, [P, P, P, I64, I64, I64, I64, D, P, P, P, P, P, P]),
    "gdt_transport_simplex_many": (I32, [I64, P, P, P, P, P, P, P, P, P, D, P, P, P, P, P, P, P,
                                         I32]),
    "gdt_transport_simplex_many_flags": (I32, [I64, P, P, P, P, P, P, P, P, P, D, P, P, P, P, P,
                                               P, P, I32, P, P]),
}

_lib = None


class NativeError(GridotError):
    """A C-ABI call failed (bad arguments or a CUDA error)."""


TORCH_EXT_PATH = os.path.join(_HERE, "csrc", "libgridot_torch.so")
_torch_ops = False


def load_torch_extension() -> bool:
    """Load the PyTorch extension (csrc/torch_ops.cpp): it brings in
    libgridot_b200.so as its linked dependency and registers
    torch.ops.gridot_b200.{version, sumpool, weighted_cost}.  Skipped when
    GRIDOT_B200_LIB selects another build of the C library."""
    global _torch_ops
    if _torch_ops or os.environ.get("GRIDOT_B200_LIB"):
        return _torch_ops
    if not os.path.exists(TORCH_EXT_PATH):
        raise NativeError(f"{TORCH_EXT_PATH} is missing; build it with "
                          "`python -m paper_2506_00976_b200.csrc.build`")
    import torch

    torch.ops.load_library(TORCH_EXT_PATH)
    _torch_ops = True
    return True


def torch_ops():
    """torch.ops.gridot_b200 (None under a GRIDOT_B200_LIB override)."""
    lib()
    if not _torch_ops:
        return None
    import torch

    return torch.ops.gridot_b200


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeError(
                f"{LIB_PATH} is missing; build it with "
                "`python -m paper_2506_00976_b200.csrc.build` (there is no CPU fallback)")
        # the C library is loaded through the PyTorch extension (its linked
        # dependency); ctypes then binds the remaining entry points on the
        # same, already loaded library
        load_torch_extension()
        handle = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGNATURES)


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().gdt_last_error().decode(errors="replace")
        raise NativeError(f"{what} failed with status {rc}: {msg}")


def ptr(t) -> int | None:
    """Raw device/host pointer of a torch tensor or numpy array (None -> NULL)."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def i64s(values) -> ctypes.Array:
    arr = (ctypes.c_int64 * len(values))(*[int(v) for v in values])
    return arr


def stream_handle(device=None) -> int:
    import torch

    return torch.cuda.current_stream(device).cuda_stream
