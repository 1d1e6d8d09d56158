"""Summaries of ncu outputs for profiles/ (development tool).

  python tools/summarize_ncu.py launches <launches.csv>          per-kernel totals + shares
  python tools/summarize_ncu.py full <report.ncu-rep>            key metrics per captured kernel
  python tools/summarize_ncu.py traffic <report.ncu-rep> <regex>  DRAM bytes summed over matching kernels
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, gi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("st::<unnamed>::", "")
        if "<" in r[ki]:
            name = r[ki].split("(CUtensor")[0].split("(float")[0].split("(const")[0].split("(int")[0]
            name = name.replace("void ", "").replace("st::<unnamed>::", "")
        key = (name[:70], r[gi])
        agg[key][0] += 1
        agg[key][1] += v
    tot = sum(v[1] for v in agg.values())
    out = ["kernel,grid,launches,total_us,avg_us,share_pct"]
    for (n, g), (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"\"{n}\",\"{g}\",{c},{t / 1e3:.1f},{t / c / 1e3:.2f},{100 * t / tot:.2f}")
    out.append(f"TOTAL,,{sum(v[0] for v in agg.values())},{tot / 1e3:.1f},,100")
    return "\n".join(out)


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active"]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")][:90]
        out.append(f"== {name}")
        for w in WANT:
            if w in h:
                j = h.index(w)
                out.append(f"   {w} = {r[j]} {units[j]}")
    return "\n".join(out)




def traffic(path, regex):
    """Σ (dram__bytes_read.sum + dram__bytes_write.sum) over captured kernels whose name
    matches `regex` (one captured step → bytes per step)."""
    import re
    if path.endswith(".csv"):
        raw = open(path).read()  # `ncu -i <rep> --page raw --csv` output
    else:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    ki, r_i, w_i, t_i = (h.index(x) for x in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                              "gpu__time_duration.sum"))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    tscale = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
    tot, tot_t, n = 0.0, 0.0, 0
    for r in rows[2:]:
        if re.search(regex, r[ki]):
            tot += float(r[r_i].replace(",", "")) * scale[units[r_i]] + float(r[w_i].replace(",", "")) * scale[units[w_i]]
            tot_t += float(r[t_i].replace(",", "")) * tscale[units[t_i]]
            n += 1
    return n, tot, tot_t


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        print(launches(sys.argv[2]))
    elif sys.argv[1] == "traffic":
        n, b, t = traffic(sys.argv[2], sys.argv[3])
        print(f"{n} kernels, dram bytes {b:.6e}, duration {t * 1e6:.1f} us")
    else:
        print(full(sys.argv[2]))
