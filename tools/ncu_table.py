"""Print per-launch ncu metrics (duration, DRAM read/write) from --csv metric logs."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader([ln for ln in open(path) if ln.startswith('"')]))
    hdr = rows[0]
    ik, im, iv, iid = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    d = collections.OrderedDict()
    for r in rows[1:]:
        d.setdefault(r[iid], {"k": r[ik]})[r[im]] = float(r[iv].replace(",", ""))
    return list(d.values())


if __name__ == "__main__":
    for path in sys.argv[1:]:
        L = load(path)
        tot = sum(v["gpu__time_duration.sum"] for v in L) / 1e6
        rd = sum(v["dram__bytes_read.sum"] for v in L) / 1e9
        print(f"{path}: total {tot:.3f} ms, read {rd:.2f} GB")
        for v in L:
            k = v["k"]
            k = k[k.find("gs_stage_kernel"):k.find("(rkb")] if "gs_stage_kernel" in k else k[:40]
            t = v["gpu__time_duration.sum"] / 1e6
            print(f"   {k:48s} {t:7.3f} ms  read {v['dram__bytes_read.sum']/1e9:6.2f} GB  write {v['dram__bytes_write.sum']/1e9:5.2f} GB")
