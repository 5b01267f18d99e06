import sys, numpy as np
sys.path.insert(0, '.')
import gpagen
from tests._common import run_gpu, run_oracle, compare
prog = gpagen.config_program(3)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3_000_000
recs = gpagen.config_stream(prog, 3).host(0, n)
g = run_gpu(prog, recs)
print("variant", g["program"].variant, "stats", g["stats"])
o = run_oracle(prog, recs)
d = (g["C"].astype(np.int64) - o["C"].astype(np.int64))
print("count diff nonzero bins", np.count_nonzero(d), "sum", d.sum())
compare(g, o)
print("PARITY OK")
