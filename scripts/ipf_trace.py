#!/usr/bin/env python
"""Phase clocks of sweep 10 of the exact fp64 IPF (ipf_kernel), pair 0.

    bash scripts/build_trace.sh
    GRIDOT_B200_LIB=paper_2506_00976_b200/csrc/_trace/libgridot_b200.so \
        python scripts/ipf_trace.py [cfg]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2506_00976_b200 as G  # noqa: E402
from paper_2506_00976_b200 import _native as N  # noqa: E402
from paper_2506_00976_b200 import synthetic as S  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
wl = S.WORKLOADS[cfg]
B = 1 if cfg == 1 else 8
mus, nus = S.batch(cfg, 0, B)
names = ["stage a", "col units", "col finish", "col cells", "stage b", "row units",
         "row finish", "row cells", "reduce"]
for rep in range(2):
    G.quantized_bounds(mus, nus, wl.dims, wl.combos[0][0], wl.combos[0][1], precision="fp64",
                       xi=0.0, max_iter=20, methods=("primal_upscaling",))
    buf = (ctypes.c_longlong * 16)()
    N.lib().gdt_debug_ex_trace(buf)
    t = np.array(buf[:10], dtype=np.int64)
    d = np.diff(t)
    print(f"cfg{cfg} sweep total {t[9] - t[0]} cycles: " +
          ", ".join(f"{n} {int(x)}" for n, x in zip(names, d)))
