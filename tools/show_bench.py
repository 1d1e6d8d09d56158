"""Print the key fields of bench JSON lines (development helper)."""
import json, sys
for f in sys.argv[1:]:
    for l in open(f):
        l = l.strip()
        if not l.startswith("{"):
            continue
        d = json.loads(l)
        r = d.get("roofline") or {}
        e = d.get("e2e") or {}
        print(f, d["config"].get("workload"), "S=%s" % d["config"].get("stages"), "value=%.0f" % d["value"],
              "ms=%.3f" % d["ms_per_step"], "frac=%s" % (r.get("frac") and round(r["frac"], 3)),
              "e2e=%s" % (e.get("value") and round(e["value"])), d.get("kernel_ms_per_step"), d["clocks"])
