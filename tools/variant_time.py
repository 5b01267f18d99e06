"""Tuning probe: time the config-3 ingest with an alternative build of the library
(`python tools/variant_time.py build/libX.so [records] [cfg]`) and check its count table against the
product library's on the same records (both GPU; the oracle parity lives in tests/)."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import gpagen
from paper_2009_04061_b200 import gpa as G

lib_path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000_000
cfg = int(sys.argv[3]) if len(sys.argv) > 3 else 3
prog = gpagen.config_program(cfg)
recs = gpagen.config_stream(prog, cfg).device(0, n)
if lib_path != "product":
    G.LIB_PATH = os.path.join(ROOT, lib_path)
P = G.Program(prog)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
reps = 1 if n >= 100_000_000 else 20   # short streams: back-to-back calls, so host launch cost hides
for it in range(8):
    P.reset()
    ev[0].record()
    for _ in range(reps):
        P.ingest(recs)
    ev[1].record(); torch.cuda.synchronize()
    if it >= 3:
        ts.append(ev[0].elapsed_time(ev[1]) / reps)
P.reset(); P.ingest(recs); torch.cuda.synchronize()
counts = P.view("counts").cpu().numpy()
out = os.path.join(ROOT, "gpurun_out", f"counts{cfg}_" + os.path.basename(lib_path) + ".npy")
os.makedirs(os.path.dirname(out), exist_ok=True)
np.save(out, counts)
ms = float(np.median(ts))
print(f"{lib_path} cfg{cfg}: ingest {ms:.4f} ms  {n * 8 / ms / 1e6:.0f} GB/s  sum={int(counts.sum())}")
