"""One config-4 step for ncu (no timing)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from gpagen import batch
from gpagen.patterns import table2
from paper_2009_04061_b200 import Program
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
prog = batch.config4_program()
recs = batch.config4_stream(prog).device(0, n).view(torch.int64)
order, sb, sk = batch.grouped_order(recs & 0xFFFFFFFF, prog)
g = recs[order]; del recs, order
sb_t = torch.from_numpy(sb.astype(np.int64)).cuda(); sk_t = torch.from_numpy(sk.view(np.int32)).cuda()
P = Program(prog); P.set_patterns(table2(prog.n_reasons))
torch.cuda.synchronize()
P.reset(); P.ingest_segments(g, sb_t, sk_t); P.blame(); P.aggregate(); P.estimate()
torch.cuda.synchronize()
