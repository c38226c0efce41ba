#!/usr/bin/env python
"""Phase clocks of sweep 10 of the coarse-level primal stage (primal_coarse_kernel), CTA 0.

    bash scripts/build_trace.sh
    GRIDOT_B200_LIB=paper_2506_00976_b200/csrc/_trace/libgridot_b200.so \
        python scripts/coarse_trace.py [cfg] [pairs]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2506_00976_b200 as G  # noqa: E402
from paper_2506_00976_b200 import _native as N  # noqa: E402
from paper_2506_00976_b200 import synthetic as S  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
pairs = int(sys.argv[2]) if len(sys.argv) > 2 else 8
wl = S.WORKLOADS[cfg]
mus, nus = S.batch(cfg, 0, pairs)
names = ["S_k pass", "matvec K^T a", "B_l pass", "matvec K b", "row pass", "reduce"]
for rep in range(2):
    G.quantized_bounds(mus, nus, wl.dims, wl.combos[0][0], wl.combos[0][1], precision="fp32",
                       xi=0.0, max_iter=20, methods=("weighted_cost", "primal_upscaling"))
    buf = (ctypes.c_longlong * 16)()
    N.lib().gdt_debug_ex_trace(buf)
    t = np.array(buf[:7], dtype=np.int64)
    print(f"cfg{cfg} x{pairs} coarse sweep {t[6] - t[0]} cycles: " +
          ", ".join(f"{n} {int(x)}" for n, x in zip(names, np.diff(t))))
