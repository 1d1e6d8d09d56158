"""Aggregate ncu warp-stall samples per CUDA source line (ncu -i X --page source --csv --print-source cuda,sass).
usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
r = list(csv.reader(out))
hdr = None
agg = {}
cur = None
for row in r:
    if len(row) > 2 and row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or len(row) < 5:
        continue
    if row[0]:
        cur = (int(row[0]), row[1].strip()[:100])
        agg.setdefault(cur, [0, 0])
        continue
    if cur is None:
        continue
    try:
        agg[cur][0] += int(row[4] or 0)
        agg[cur][1] += int(row[7] or 0)
    except ValueError:
        pass
tot = sum(v[0] for v in agg.values())
print("total samples", tot)
for (ln, src), (smp, ie) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{smp:6d} {100.0 * smp / max(tot, 1):5.1f}% {ie:10d}  L{ln}: {src}")
