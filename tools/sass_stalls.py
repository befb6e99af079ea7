"""Top SASS lines by warp-stall samples of each kernel in an .ncu-rep (source page).
    python tools/sass_stalls.py report.ncu-rep [n_lines]"""
import csv
import io
import subprocess
import sys
from collections import Counter


def main(path, nl=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks, cur = [], None
    for r in csv.reader(io.StringIO(out)):
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            blocks.append(cur)
        elif r and r[0] == "Address":
            cur["hdr"] = r
        elif cur is not None and r:
            cur["rows"].append(r)
    for b in blocks:
        ix = {k: i for i, k in enumerate(b["hdr"])}
        sc = [k for k in b["hdr"] if k.startswith("stall_") and "Not Issued" not in k]
        tot, op, data = Counter(), Counter(), []
        for r in b["rows"]:
            s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
            st = {k: int(r[ix[k]] or 0) for k in sc}
            tot.update(st)
            src = r[ix["Source"]]
            o = (src.split()[1] if src.startswith("@") else src.split()[0]).split(".")[0] if src.split() else "?"
            op[o] += s
            data.append((s, src, st))
        T = sum(d[0] for d in data)
        print("==", b["name"][:120], "samples", T)
        print("   stalls:", ", ".join(f"{k[6:]}={v / T:.1%}" for k, v in tot.most_common(8)))
        print("   opcodes:", ", ".join(f"{k}={v / T:.1%}" for k, v in op.most_common(12)))
        for s, src, st in sorted(data, key=lambda x: -x[0])[:nl]:
            top = ", ".join(f"{k[6:]}={v}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:2])
            print(f"   {s / T:6.2%}  {src[:64]:64s} {top}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
