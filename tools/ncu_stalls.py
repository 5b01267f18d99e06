"""Top stall PCs of an ncu source page with their stall-reason breakdown, plus per-region totals.
usage: python tools/ncu_stalls.py report.ncu-rep [n_top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
f = lambda x: float(x.replace(',', '') or 0)
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(f(r[ix["Warp Stall Sampling (All Samples)"]]) for r in data) or 1
agg = {k: sum(f(r[ix[k]]) for r in data) for k in reasons}
print("all stall samples by reason:", ", ".join(f"{k[6:]} {100 * v / tot:.1f}%" for k, v in
                                                 sorted(agg.items(), key=lambda x: -x[1]) if v / tot > 0.005))
top = sorted(data, key=lambda r: -f(r[ix["Warp Stall Sampling (All Samples)"]]))[:ntop]
for r in top:
    s = f(r[ix["Warp Stall Sampling (All Samples)"]])
    rs = sorted(((k[6:], f(r[ix[k]])) for k in reasons), key=lambda x: -x[1])[:3]
    print(f"{r[ix['Address']][-5:]} {100 * s / tot:5.1f}%  {r[ix['Source']][:58]:58s} " +
          " ".join(f"{k}:{100 * v / s:.0f}%" for k, v in rs if v))
