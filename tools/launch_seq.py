"""Print the per-launch sequence (duration, grid, kernel) of the last N launches of an
ncu --csv launch list (development tool)."""
import csv
import sys
from collections import OrderedDict

path, n = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 200
rows = list(csv.reader(open(path)))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi, gi, mi, ii = (h.index(x) for x in ("Kernel Name", "Metric Value", "Grid Size", "Metric Name", "ID"))
d = OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    d.setdefault(r[ii], {"name": r[ki], "grid": r[gi]})[r[mi]] = float(r[vi].replace(",", ""))
L = list(d.values())
tot = 0.0
for e in L[-n:]:
    nm = e["name"].replace("void ", "").replace("st::<unnamed>::", "")
    nm = nm.split("(CUtensor")[0].split("(float")[0].split("(const")[0][:64]
    t = e.get("gpu__time_duration.sum", 0) / 1e3
    tot += t
    extra = ""
    if "dram__bytes_read.sum" in e:
        extra = f"{e['dram__bytes_read.sum'] / 1e6:8.1f} {e.get('dram__bytes_write.sum', 0) / 1e6:8.1f} MB"
    print(f"{t:8.1f} us {extra} {e['grid']:>14} {nm}")
print(f"total {tot:.1f} us over {min(n, len(L))} launches")
