"""Host-LP thread scaling probe: serial vs all cores on cfg3 C-tilde LPs."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2506_00976_b200 import synthetic as S
from paper_2506_00976_b200.exact import build_transport_problem, solve_transport_many
from paper_2506_00976_b200.costs import centre_cost_table
from paper_2506_00976_b200.measures import GridSpec

def sumpool(x, dims, k):
    a = x.reshape(tuple(reversed(dims)))
    n1, n0 = dims[1] // k, dims[0] // k
    return a.reshape(n1, k, n0, k).sum(axis=(1, 3)).reshape(-1)

B = 45
mus, nus = S.batch(3, 0, B)
dims = (128, 128)
for k, p in [(4, 1.0), (4, 2.0)]:
    T = centre_cost_table(dims, k, p)
    probs = [build_transport_problem(sumpool(mus[b], dims, k), sumpool(nus[b], dims, k), T) for b in range(B)]
    t = time.perf_counter(); solve_transport_many(probs[:8], threads=1, slack=False); ser = (time.perf_counter() - t) / 8
    for th in (4, 8, 16):
        t = time.perf_counter(); solve_transport_many(probs, threads=th, slack=False); par = time.perf_counter() - t
        print(f"k{k} p{p}: serial {ser:.3f} s/LP; {th} threads: {par:.3f} s for {B} LPs -> efficiency {B * ser / th / par:.2f}", flush=True)
