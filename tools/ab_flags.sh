#!/bin/bash
# A/B of compile-time kernel knobs (rk_pair.cu: RKB_PAIR_EARLY, RKB_RING_WARPS, RKB_PAIR_RMAX ...):
# rebuilds rk_pair.cu with each flag set, runs the adaptive + rk4 legs, prints per-role times.
# usage (on the GPU box): bash tools/ab_flags.sh "-DRKB_PAIR_EARLY=0" "-DRKB_PAIR_EARLY=1" ...
# ("base" = no extra flag)
i=0
for f in "$@"; do
  i=$((i + 1))
  [ "$f" = base ] && f=""
  touch paper_2309_05331_b200/csrc/rk_pair.cu
  RKB_NVCC_EXTRA="$f" python -m paper_2309_05331_b200.build > gpurun_out/ab_build_$i.log 2>&1 || { echo "build failed: $f"; continue; }
  timeout 600 python bench.py --legs ${AB_LEGS:-adaptive,rk4} --steps 10 > gpurun_out/ab_$i.json 2>/dev/null
  python - "$f" gpurun_out/ab_$i.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
r = d["roofline"]["kernels"]
x = d.get("extra", {}).get("rk4", {})
print(f"{sys.argv[1] or 'base':28s} try {d['config']['ms_per_try']:.3f}",
      " ".join(f"{k} {v['avg_launch_ms']:.3f}" for k, v in r.items()),
      f"rk4 {x.get('ms_per_step', float('nan')):.3f}", d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
done
