#!/usr/bin/env python
"""Dependent-DADD latency (cycles per add of an exact-order chain), csrc/probes.cu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2506_00976_b200 import _native as N  # noqa: E402

out = torch.zeros(1, dtype=torch.int64, device="cuda")
for adds in (1024, 8192, 65536):
    for _ in range(3):
        N.check(N.lib().gdt_probe_dadd_chain(adds, N.ptr(out), None), "probe")
        torch.cuda.synchronize()
    print(f"dadd chain: {adds} adds, {int(out[0])} cycles, {int(out[0]) / adds:.2f} cycles/add")
