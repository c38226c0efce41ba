#!/usr/bin/env python
"""Fraction of source tiles the pruned fp32 p=1 c-transform evaluates exactly.

    bash scripts/build_trace.sh
    GRIDOT_B200_LIB=paper_2506_00976_b200/csrc/_trace/libgridot_b200.so \
        python scripts/ct_trace.py

Runs the dual bound (two c-transforms per pair) of the cfg3 batch at kappa 4
and 8, p = 1, fp32 mode, and prints the tiles evaluated / brute-force tiles
(regions x 256 per transform); the executed-candidate rate of the kernel is
the brute-force-equivalent rate times this fraction.
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_00976_b200 as G  # noqa: E402
from paper_2506_00976_b200 import _native as N  # noqa: E402
from paper_2506_00976_b200 import synthetic as S  # noqa: E402

wl = S.WORKLOADS[3]
mus, nus = S.batch(3, 0, 45)
res = {}
for k in (4, 8):
    G.quantized_bounds(mus, nus, wl.dims, k, 1.0, precision="fp32", methods=("dual_upscaling",))
    buf = (ctypes.c_ulonglong * 2)()
    N.lib().gdt_debug_ct_tiles(buf, 1)
    G.quantized_bounds(mus, nus, wl.dims, k, 1.0, precision="fp32", methods=("dual_upscaling",))
    N.lib().gdt_debug_ct_tiles(buf, 0)
    regions = 45 * (128 // 16) ** 2
    brute = 2 * regions * 256  # two transforms per pair
    res[f"k{k}_p1"] = {"evaluated_tiles": buf[0], "visited_tiles": buf[1],
                       "brute_force_tiles": brute, "evaluated_fraction": buf[0] / brute}
print(json.dumps(res))
