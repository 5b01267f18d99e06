"""Per-kernel table of an ncu --csv launch list (time, DRAM bytes): python tools/launches_table.py file.csv [filter]"""
import csv, sys
from collections import OrderedDict
rows = list(csv.reader(open(sys.argv[1])))
flt = sys.argv[2] if len(sys.argv) > 2 else "gpa"
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
k, mn, v, idc = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = OrderedDict()
for r in rows[hi + 1:]:
    full = r[k].split("(")[0]
    name = full.replace("gpa::<unnamed>::", "")   # template arguments may repeat the namespace
    name = ("gpa::" + name if "gpa::" in full else name)
    name = name[:34] if "part" in name else name[-34:]   # keep the kernel name of the long template ids
    per.setdefault((r[idc], name, flt in full), {})[r[mn]] = float(r[v].replace(",", ""))
tot = 0.0
for (i, name, keep), m in per.items():
    if not keep:
        continue
    t = m.get("gpu__time_duration.sum", 0) / 1e3
    tot += t
    rd, wr = m.get("dram__bytes_read.sum", 0) / 1e6, m.get("dram__bytes_write.sum", 0) / 1e6
    print(f"{i:>4} {name:36s} {t:9.1f} us  rd {rd:9.1f} MB  wr {wr:9.1f} MB  {(rd + wr) / max(t, 1e-9):6.2f} TB/s")
print(f"total {tot:.1f} us")
