"""Turn tools/profile_round.sh outputs (gpurun_out/TAG_*) into the files committed under
profiles/: TAG_launches.{csv,txt}, TAG_warm_dram.txt, TAG_{adaptive,rk4}_full_summary.txt,
TAG_bench.json and ncu_traffic.json (cold-L2 dram bytes per stage launch of every leg, read by
bench.py for roofline.traffic).  Runs on the GPU box (ncu -i needs the .ncu-rep files).

    python tools/make_profiles.py TAG [--out DIR]     (default DIR: profiles/)
"""
import csv
import json
import os
import shutil
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import summarize_ncu as sn  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def full_launch_bytes(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(m)
            b += float(r[i].replace(",", "")) * SCALE.get(units[i], 1.0)
        out.append([r[hdr.index("Kernel Name")], b])
    return out


def csv_launch_bytes(path):
    per = {}
    order = []
    for d in sn.read_csv_rows(path):
        key = (d["ID"], d["Kernel Name"])
        if key not in per:
            per[key] = 0.0
            order.append(key)
        if d["Metric Name"] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            per[key] += float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1.0)
    return [[k[1], per[k]] for k in order]


def main(tag, out):
    g = os.path.join(ROOT, "gpurun_out")
    os.makedirs(out, exist_ok=True)
    shutil.copy(os.path.join(g, f"{tag}_launches.csv"), os.path.join(out, f"{tag}_launches.csv"))
    open(os.path.join(out, f"{tag}_launches.txt"), "w").write(sn.launches(os.path.join(g, f"{tag}_launches.csv")) + "\n")
    open(os.path.join(out, f"{tag}_warm_dram.txt"), "w").write(sn.warm(os.path.join(g, f"tune_{tag}.csv")) + "\n")
    traffic = {"_source": f"{tag} (tools/profile_round.sh): dram__bytes_read.sum + dram__bytes_write.sum per "
                          "stage launch of one step, cold L2 (ncu default cache control); adaptive (one "
                          "DOPRI5 try: the K8 head pair, K3 stages 4 and 5, the K8 tail pair), rk4 (K8, 2 launches) and rk4_k3 from ncu --set full captures, the other legs "
                          "from metrics-only captures; abm legs: the PEC launch plus rk4's k1-type launch"}
    rk4_first = None
    for leg in ("adaptive", "rk4", "rk4_k3"):
        rep = os.path.join(g, f"{tag}_full_{leg}.ncu-rep")
        if not os.path.exists(rep):
            print("missing", rep)
            continue
        open(os.path.join(out, f"{tag}_{leg}_full_summary.txt"), "w").write(sn.full(rep) + "\n")
        pl = full_launch_bytes(rep)
        if leg == "rk4_k3":
            rk4_first = pl[0]  # the k1-type K3 stage (abm legs)
        traffic["dopri5_adaptive" if leg == "adaptive" else leg] = {
            "bytes_per_launch": sum(b for _, b in pl) / len(pl), "launches": len(pl), "per_launch": pl}
    for f in sorted(os.listdir(g)):
        if not (f.startswith(f"{tag}_dram_") and f.endswith(".csv")):
            continue
        leg = f[len(f"{tag}_dram_"):-4]
        pl = csv_launch_bytes(os.path.join(g, f))
        if not pl:
            print("empty", f)
            continue
        if leg.startswith("abm") and rk4_first:
            pl = [rk4_first] + pl
        traffic[leg] = {"bytes_per_launch": sum(b for _, b in pl) / len(pl), "launches": len(pl), "per_launch": pl}
    json.dump(traffic, open(os.path.join(out, "ncu_traffic.json"), "w"), indent=1)
    line = [l for l in open(os.path.join(g, f"{tag}_bench.log")).read().splitlines() if l.startswith("{")][-1]
    json.dump(json.loads(line), open(os.path.join(out, f"{tag}_bench.json"), "w"), indent=1)
    print("written", tag, "->", out)


if __name__ == "__main__":
    tag = sys.argv[1]
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else os.path.join(ROOT, "profiles")
    main(tag, out)
