"""Print leg / value / roofline fraction / ms from a bench.py log (JSON lines)."""
import json
import sys

for line in open(sys.argv[1]):
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    if "metric" in d:
        print("headline", "%.4g" % d["value"], "%.3f" % (d["roofline"]["frac"] or 0), "%.3f ms" % d["ms_per_step"])
    for k, v in (d.get("extra") or {}).items():
        if isinstance(v, dict) and "value" in v:
            fr = (v.get("roofline") or {}).get("frac")
            print(k, "%.4g" % v["value"], "%.3f" % (fr or 0), "%.3f ms" % v.get("ms_per_step", 0))
