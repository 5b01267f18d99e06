"""Tuning probe: median time of the analysis graph (gpa_analyze: blame + rollup + estimate) for
configs 2 and 3 with an alternative build of the library
(`python tools/analyze_time.py lib|product [2,3,4] [auto|graph|fused]`)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import gpagen
from gpagen.patterns import table2
from paper_2009_04061_b200 import gpa as G

lib_path = sys.argv[1]
if lib_path != "product":
    G.LIB_PATH = os.path.join(ROOT, lib_path)
from gpagen import batch
cfgs = [int(c) for c in sys.argv[2].split(",")] if len(sys.argv) > 2 else [2, 3]
mode = sys.argv[3] if len(sys.argv) > 3 else "auto"
nopat = len(sys.argv) > 4 and sys.argv[4] == "nopat"   # blame + rollup only (no estimate branch)
out = []
for cfg in cfgs:
    if cfg == 4:    # the batch program; plain ingest gives the same counts as the segment ingest
        prog = batch.config4_program()
        recs = batch.config4_stream(prog).device(0, 100_000_000)
    else:
        prog = gpagen.config_program(cfg)
        recs = gpagen.config_stream(prog, cfg).device(0, {2: 10_000_000, 3: 100_000_000}[cfg])
    P = G.Program(prog)
    if not nopat:
        P.set_patterns(table2(prog.n_reasons))
    P.analyze_mode = mode
    P.reset(); P.ingest(recs)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ts = []
    for it in range(25):
        ev[0].record(); P.analyze(); ev[1].record(); torch.cuda.synchronize()
        if it >= 5:
            ts.append(ev[0].elapsed_time(ev[1]))
    if nopat:
        out.append(f"cfg{cfg} analyze(no patterns) {np.median(ts) * 1e3:.1f} us")
        continue
    est = P.read_estimates_array()
    np.save(os.path.join(ROOT, "gpurun_out", f"est_{cfg}_{os.path.basename(lib_path)}_{mode}.npy"),
            np.stack([est["speedup"], est["M"]]))
    out.append(f"cfg{cfg} analyze {np.median(ts) * 1e3:.1f} us")
print(lib_path + f" [{mode}]: " + "  ".join(out))
