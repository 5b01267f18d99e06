"""Probe: backward slicing of a large random SASS program on the GPU (gpa_slice) vs the oracle."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from gpagen import sass
from paper_2009_04061_b200 import slice_sass
n_funcs = int(sys.argv[1]) if len(sys.argv) > 1 else 600
S = sass.random_sass(n_funcs, 99)
print("instructions", S.n_instr, "blocks", len(S.block_begin) - 1)
slice_sass(S)                      # warm-up (module load)
tgs = []
for _ in range(5):
    t = time.perf_counter(); g = slice_sass(S); tgs.append(time.perf_counter() - t)
tg = sorted(tgs)[2]   # median of 5 calls
t = time.perf_counter(); o = oracle.slice_program(S); to = time.perf_counter() - t
same = all(np.array_equal(g[k], o[k]) for k in g)
print(f"edges {len(g['edge_def'])}  gpu {tg*1e3:.1f} ms  oracle {to*1e3:.1f} ms  identical {same}")
