"""Print leg / value / roofline fraction / ms from a bench.py log (JSON lines)."""
import json
import sys

for line in open(sys.argv[1]):
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    if "metric" in d:
        print("headline", "%.4g" % d["value"], "%.3f" % (d["roofline"]["frac"] or 0), "%.3f ms" % d["ms_per_step"])
    if "e2e" in d:
        print("e2e", "%.4g" % d["e2e"]["value"])
    for k, v in (d.get("extra") or {}).items():
        if not isinstance(v, dict):
            continue
        if "value" in v:
            fr = (v.get("roofline") or {}).get("frac") or v.get("frac_of_peak") or 0
            print(k, "%.4g" % v["value"], "%.3f" % fr, "%.3f ms" % v.get("ms_per_step", 0))
        for m, w in v.items():
            if isinstance(w, dict) and "value" in w:
                print(f"{k}.{m}", "%.4g" % w["value"], "%.4f ms" % w.get("ms_per_step", 0),
                      "launches/step %.3g" % w.get("gpu_launches_per_step", 0))
