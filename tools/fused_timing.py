"""Tuning probe: per-phase times of the fused analysis kernel as CTA 0 sees them (build/libft.so,
built with -DGPA_FUSED_TIMING): `python tools/fused_timing.py [cfg] [grid]`."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import gpagen
from gpagen.patterns import table2
from paper_2009_04061_b200 import gpa as G

G.LIB_PATH = os.environ.get("GPA_FT_LIB") or os.path.join(ROOT, "build", "libft.so")
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
if len(sys.argv) > 2:
    os.environ["GPA_FUSED_GRID"] = sys.argv[2]
prog = gpagen.config_program(cfg)
recs = gpagen.config_stream(prog, cfg).device(0, 10_000_000)
P = G.Program(prog)
P.set_patterns(table2(prog.n_reasons))
P.analyze_mode = "fused"
P.reset(); P.ingest(recs)
buf = (ctypes.c_ulonglong * 16)()
rows = []
for it in range(20):
    P.analyze(); torch.cuda.synchronize()
    G.lib().gpa_debug_fused_timing(buf)
    t = np.array(buf[:], dtype=np.int64)
    if it >= 5:
        rows.append(np.diff(t[[0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 15]]) / 1e3)
m = np.median(np.array(rows), axis=0)
names = ["blame", "sync", "def+est", "sync", "tiles+seg1", "sync", "rseg1+seg2", "sync", "rseg2", "sync", "final"]
print(f"cfg{cfg} grid={os.environ.get('GPA_FUSED_GRID', 'auto')}: " + "  ".join(f"{n} {v:.1f}" for n, v in zip(names, m)),
      f"total {m.sum():.1f} us")
