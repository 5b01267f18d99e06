"""Per-region (split at barriers / mbarrier waits) instruction and stall shares of an ncu source page."""
import csv, subprocess, sys, io
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]; data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
f = lambda x: float(x.replace(',', '') or 0)
tot_s = sum(f(r[ix['Warp Stall Sampling (All Samples)']]) for r in data) or 1
tot_e = sum(f(r[ix['Instructions Executed']]) for r in data) or 1
if len(sys.argv) > 2:
    with open(sys.argv[2], 'w') as fh:
        for r in data:
            fh.write(f"{r[ix['Address']][-5:]} {f(r[ix['Instructions Executed']]):>10.0f} {100*f(r[ix['Warp Stall Sampling (All Samples)']])/tot_s:>6.2f}  {r[ix['Source']]}\n")
cur = None; acc = []
for r in data:
    src = r[ix['Source']]; a = r[ix['Address']][-5:]
    if cur is None or 'BAR.SYNC' in src or 'SYNCS.PHASECHK' in src:
        if cur: acc.append(cur)
        cur = [a, 0, 0, src.strip()[:40]]
    cur[1] += f(r[ix['Instructions Executed']]); cur[2] += f(r[ix['Warp Stall Sampling (All Samples)']])
acc.append(cur)
print('total warp-instructions executed', tot_e)
for a in acc:
    if a[1] / tot_e > 0.005 or a[2] / tot_s > 0.01:
        print(a[0], 'exec %.1f%%' % (100 * a[1] / tot_e), 'stall %.1f%%' % (100 * a[2] / tot_s), a[3])
top = sorted(data, key=lambda r: -f(r[ix['Warp Stall Sampling (All Samples)']]))[:10]
for r in top:
    print('  ', r[ix['Address']][-5:], r[ix['Source']][:70], '%.1f%%' % (100 * f(r[ix['Warp Stall Sampling (All Samples)']]) / tot_s))
