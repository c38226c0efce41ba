#!/usr/bin/env python
"""Phase clocks of sweep 10 of the clustered exact IPF (ipf_cluster_kernel), CTA 0.

    bash scripts/build_trace.sh
    GRIDOT_B200_LIB=paper_2506_00976_b200/csrc/_trace/libgridot_b200.so \
        python scripts/ipf_cl_trace.py [cfg] [pairs] [cluster size]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
pairs = int(sys.argv[2]) if len(sys.argv) > 2 else 64
if len(sys.argv) > 3:
    os.environ["GRIDOT_IPF_CLUSTER"] = sys.argv[3]

import paper_2506_00976_b200 as G  # noqa: E402
from paper_2506_00976_b200 import _native as N  # noqa: E402
from paper_2506_00976_b200 import synthetic as S  # noqa: E402

wl = S.WORKLOADS[cfg]
mus, nus = S.batch(cfg, 0, pairs)
names = ["col units", "col cells", "flags + barrier C", "row units", "row cells",
         "reduce + barrier A"]
for rep in range(2):
    G.quantized_bounds(mus, nus, wl.dims, wl.combos[0][0], wl.combos[0][1], precision="fp64",
                       xi=0.0, max_iter=20, methods=("primal_upscaling",))
    buf = (ctypes.c_longlong * 16)()
    N.lib().gdt_debug_ex_trace(buf)
    t = np.array(buf[:7], dtype=np.int64)
    d = np.diff(t)
    print(f"cfg{cfg} x{pairs} cluster {os.environ.get('GRIDOT_IPF_CLUSTER', 'auto')}: sweep "
          f"{t[6] - t[0]} cycles: " + ", ".join(f"{n} {int(x)}" for n, x in zip(names, d)))
    u = np.array(buf[8:13], dtype=np.int64)
    print("   first col batch: " + ", ".join(f"{n} {int(x)}" for n, x in zip(
        ["products", "barrier", "chains (thread 0)", "barrier"], np.diff(u))))
