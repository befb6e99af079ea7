"""Per-launch table (ms, DRAM GB, GB/s, L2 hit, warps active) from a tools/tune.sh ncu csv."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
per = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    key = (d["ID"], d["Kernel Name"])
    per.setdefault(key, {})[d["Metric Name"]] = (float(d["Metric Value"].replace(",", "")), d["Metric Unit"])
for (i, name), m in per.items():
    t = m["gpu__time_duration.sum"]
    ms = t[0] / 1e6 if t[1] in ("ns", "nsecond") else (t[0] / 1e3 if t[1] in ("us", "usecond") else t[0])

    def gb(k):
        v, u = m[k]
        return v * {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3}.get(u, 1e-9)
    rd, wr = gb("dram__bytes_read.sum"), gb("dram__bytes_write.sum")
    print("%-40s %7.3f ms  rd %6.2f wr %6.2f GB  %5.0f GB/s  L2hit %5.1f  warps %5.1f" % (
        name.split("::")[-1][:40], ms, rd, wr, (rd + wr) / ms * 1e3,
        m["lts__t_sector_hit_rate.pct"][0], m["sm__warps_active.avg.pct_of_peak_sustained_active"][0]))
