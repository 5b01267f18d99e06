"""Summarise an ncu report: key metrics + top stall sites (source page). Usage: python tools/ncu_summary.py rep [n]"""
import csv, io, subprocess, sys

def page(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))

def details(rep):
    rows = page(rep, "--page", "details")
    hdr = rows[0]
    res = []
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        res.append((d.get("Kernel Name", "")[:60], d.get("Section Name", ""), d.get("Metric Name", ""), d.get("Metric Value", ""), d.get("Metric Unit", "")))
    return res

def raw(rep, names):
    rows = page(rep, "--page", "raw")
    hdr, units, vals = rows[0], rows[1], rows[2:]
    out = []
    for v in vals:
        d = dict(zip(hdr, v))
        out.append({n: d.get(n) for n in names})
    return out

def src(rep, n=20):
    rows = page(rep, "--page", "source", "--print-source", "sass")
    hdr = rows[1]; data = rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    f = lambda x: float(x.replace(",", "") or 0)
    tot = sum(f(r[ix["Warp Stall Sampling (All Samples)"]]) for r in data) or 1
    top = sorted(data, key=lambda r: -f(r[ix["Warp Stall Sampling (All Samples)"]]))[:n]
    return [(r[ix["Address"]][-5:], r[ix["Source"]][:80], round(100 * f(r[ix["Warp Stall Sampling (All Samples)"]]) / tot, 1), r[ix["Instructions Executed"]]) for r in top]

if __name__ == "__main__":
    rep = sys.argv[1]
    keys = {"Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput", "Compute (SM) Throughput", "Executed Ipc Active", "Issued Instructions", "Registers Per Thread", "Achieved Occupancy", "L2 Hit Rate", "One or More Eligible", "Warp Cycles Per Issued Instruction"}
    for k, s, m, v, u in details(rep):
        if m in keys:
            print(f"{m:40s} {v} {u}")
    for d in raw(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "gpu__time_duration.sum"]):
        print(d)
    for row in src(rep, int(sys.argv[2]) if len(sys.argv) > 2 else 20):
        print(*row)
