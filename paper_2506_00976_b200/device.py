"""Device plumbing: CUDA device selection, host<->device moves, stream handle.

PyTorch supplies device memory (caching allocator), streams and
torch.distributed; every hot-path computation runs in libgridot_b200.so.
There is no CPU execution path: without a CUDA device these helpers raise.
"""

from __future__ import annotations

import numpy as np

from ._native import lib, stream_handle
from .errors import GridotError

_torch = None


class NoDeviceError(GridotError):
    """A CUDA device is required for this operation and none is visible."""


def torch():
    global _torch
    if _torch is None:
        import torch as _t

        _torch = _t
    return _torch


def device():
    t = torch()
    if not t.cuda.is_available():
        raise NoDeviceError("paper_2506_00976_b200 needs a CUDA device (B200, sm_100a); "
                            "there is no CPU fallback")
    lib()  # fail loudly if the native library is missing
    return t.device("cuda", t.cuda.current_device())


def to_dev(a, dtype=None):
    """numpy / torch -> contiguous CUDA tensor (float64 unless dtype given)."""
    t = torch()
    dev = device()
    if isinstance(a, t.Tensor):
        out = a.to(dev, non_blocking=True)
    else:
        arr = np.ascontiguousarray(a)
        if not arr.flags.writeable:
            arr = arr.copy()
        out = t.from_numpy(arr).to(dev, non_blocking=True)
    if dtype is not None:
        out = out.to(dtype)
    return out.contiguous()


def to_host(t):
    return t.detach().cpu().numpy()


def pinned_empty(shape, dtype=None):
    """A fresh page-locked host buffer of `shape` (float64 by default) from
    torch's caching host allocator; returns (torch view, numpy view) aliasing
    it.  The numpy view keeps the buffer alive; nothing is shared between
    callers."""
    tt = torch()
    buf = tt.empty(tuple(shape), dtype=dtype or tt.float64, pin_memory=True)
    return buf, buf.numpy()


def to_host_pinned(t):
    """D2H through a fresh page-locked buffer (full PCIe/NVLink-C2C rate);
    returns a numpy array that owns (keeps alive) the buffer."""
    tt = torch()
    buf, arr = pinned_empty(t.shape, t.dtype)
    buf.copy_(t.detach(), non_blocking=True)
    tt.cuda.current_stream(t.device).synchronize()
    return arr


def stream() -> int:
    return stream_handle(device())
