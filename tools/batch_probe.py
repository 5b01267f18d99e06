"""Probe: config 4 (batch of 10^4 kernels) step breakdown on one GPU."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from gpagen import batch
from gpagen.patterns import table2
from paper_2009_04061_b200 import Program

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
t = time.time(); prog = batch.config4_program(); print("gen", time.time() - t, flush=True)
spec = batch.config4_stream(prog)
recs = spec.device(0, n).view(torch.int64)
order, sb, sk = batch.grouped_order(recs & 0xFFFFFFFF, prog)
g = recs[order]
del recs, order
sb_t = torch.from_numpy(sb.astype(np.int64)).cuda(); sk_t = torch.from_numpy(sk.view(np.int32)).cuda()
t = time.time(); P = Program(prog); print("create", time.time() - t, "segments", len(sk), flush=True)
P.set_patterns(table2(prog.n_reasons))
s = torch.cuda.current_stream()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
for it in range(5):
    ev[0].record(s); P.reset(); ev[1].record(s); P.ingest_segments(g, sb_t, sk_t); ev[2].record(s)
    P.blame(); ev[3].record(s); P.aggregate(); ev[4].record(s); P.estimate(); ev[5].record(s)
    torch.cuda.synchronize()
    print("reset %.3f ingest %.3f blame %.3f aggregate %.3f estimate %.3f ms" % tuple(ev[i].elapsed_time(ev[i + 1]) for i in range(5)))
for it in range(3):
    ev[0].record(s); P.reset(); P.ingest_segments(g, sb_t, sk_t); ev[1].record(s); P.analyze(); ev[2].record(s)
    torch.cuda.synchronize()
    print("reset+ingest %.3f analyze(graph) %.3f ms" % (ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])))
# plain (ungrouped) ingest for comparison
P.reset(); ev[0].record(s); P.ingest(g); ev[1].record(s); torch.cuda.synchronize()
print("variant", P.variant, "plain ingest of the grouped stream %.3f ms" % ev[0].elapsed_time(ev[1]))
