"""Probe: config-4 segment ingest time with the library at GPA_LIB_PATH (tuning builds)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from gpagen import batch
from paper_2009_04061_b200 import Program
prog = batch.config4_program()
recs = batch.config4_stream(prog).device(0, 100_000_000).view(torch.int64)
order, sb, sk = batch.grouped_order(recs & 0xFFFFFFFF, prog)
g = recs[order].contiguous(); del recs, order
sb_t = torch.from_numpy(sb.astype(np.int64)).cuda(); sk_t = torch.from_numpy(sk.view(np.int32)).cuda()
P = Program(prog)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for it in range(6):
    P.reset(); ev[0].record(); P.ingest_segments(g, sb_t, sk_t); ev[1].record(); torch.cuda.synchronize()
    if it >= 2: ts.append(ev[0].elapsed_time(ev[1]))
C = P.view("counts").sum().item()
print(os.environ.get("GPA_LIB_PATH", "product"), "segment ingest %.3f ms" % np.median(ts), "sum", C)
