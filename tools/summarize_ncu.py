"""Summarise ncu outputs (gpurun_out/) into committed text files under profiles/.

    python tools/summarize_ncu.py <launches.csv> <warm.csv> <full.ncu-rep> <bench.log> <tag>
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def read_csv_rows(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            yield dict(zip(hdr, r))


def to_ms(v, unit):
    v = float(v)
    return {"ns": v / 1e6, "nsecond": v / 1e6, "us": v / 1e3, "usecond": v / 1e3, "ms": v,
            "msecond": v}.get(unit, v)


def launches(path):
    agg = collections.OrderedDict()
    tot = 0.0
    for d in read_csv_rows(path):
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        ms = to_ms(d["Metric Value"], d["Metric Unit"])
        a = agg.setdefault(d["Kernel Name"], [0, 0.0, d["Grid Size"], d["Block Size"]])
        a[0] += 1
        a[1] += ms
        tot += ms
    out = ["# ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)",
           f"# total {tot:.3f} ms over {sum(a[0] for a in agg.values())} launches",
           "launches  total_ms  share  avg_ms  grid  block  kernel"]
    for k, (n, ms, g, b) in agg.items():
        out.append(f"{n:8d} {ms:9.3f} {100 * ms / tot:5.1f}% {ms / n:7.3f}  {g} {b}  {k}")
    return "\n".join(out)


def warm(path):
    per = collections.OrderedDict()
    for d in read_csv_rows(path):
        key = (d["ID"], d["Kernel Name"])
        per.setdefault(key, {})[d["Metric Name"]] = (d["Metric Value"], d["Metric Unit"])
    out = ["# ncu --cache-control none --clock-control none (warm L2, one pass per launch)",
           "kernel  ms  dram_read_GB  dram_write_GB  achieved_GB/s  l2_hit%  warps_active%"]
    for (i, k), m in per.items():
        ms = to_ms(*m["gpu__time_duration.sum"])
        rd = float(m["dram__bytes_read.sum"][0]) / 1e9
        wr = float(m["dram__bytes_write.sum"][0]) / 1e9
        out.append(f"{k}  {ms:.3f}  {rd:.3f}  {wr:.3f}  {(rd + wr) / ms * 1e3:.0f}  "
                   f"{m['lts__t_sector_hit_rate.pct'][0]}  "
                   f"{m['sm__warps_active.avg.pct_of_peak_sustained_active'][0]}")
    return "\n".join(out)


FULL_METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
                "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                "sm__warps_active.avg.pct_of_peak_sustained_active",
                "smsp__issue_active.avg.pct_of_peak_sustained_active",
                "launch__registers_per_thread", "launch__occupancy_limit_registers",
                "launch__occupancy_limit_shared_mem", "lts__t_sector_hit_rate.pct",
                "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
                "smsp__inst_executed.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    out = ["# ncu --set full --clock-control none (cold L2 per replay); key metrics per launch"]
    for r in rows[2:]:
        out.append(f"== {r[hdr.index('Kernel Name')]}")
        for m in FULL_METRICS:
            if m in hdr:
                out.append(f"   {m} = {r[hdr.index(m)]} {units[hdr.index(m)]}")
        st = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
                try:
                    st.append((float(r[i]), h.replace("smsp__average_warps_issue_stalled_", "")
                               .replace("_per_issue_active.ratio", "")))
                except ValueError:
                    pass
        out.append("   top stalls (warps per issue): " +
                   ", ".join(f"{n}={v:.2f}" for v, n in sorted(st, reverse=True)[:6]))
    return "\n".join(out)


if __name__ == "__main__":
    lc, wc, rep, bench, tag = sys.argv[1:6]
    d = os.path.join(ROOT, "profiles")
    os.makedirs(d, exist_ok=True)
    open(os.path.join(d, f"{tag}_launches.txt"), "w").write(launches(lc) + "\n")
    open(os.path.join(d, f"{tag}_warm_dram.txt"), "w").write(warm(wc) + "\n")
    open(os.path.join(d, f"{tag}_full_summary.txt"), "w").write(full(rep) + "\n")
    line = [l for l in open(bench).read().splitlines() if l.startswith("{")][-1]
    json.dump(json.loads(line), open(os.path.join(d, f"{tag}_bench.json"), "w"), indent=1)
    print("written", tag)
