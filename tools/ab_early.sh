#!/bin/bash
# A/B of rk_pair.cu's RKB_PAIR_EARLY (ring slot released one plane early): rebuilds rk_pair.cu per value,
# runs the adaptive + rk4 legs.  usage (on the GPU box): AB_VALUES="2 0 2 0" bash tools/ab_early.sh
for e in ${AB_VALUES:-2 0 2 0}; do
  touch paper_2309_05331_b200/csrc/rk_pair.cu
  RKB_NVCC_EXTRA=-DRKB_PAIR_EARLY=$e python -m paper_2309_05331_b200.build > /dev/null 2>&1
  timeout 600 python bench.py --legs adaptive,rk4 --steps 10 > gpurun_out/ab_$e.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$e.json').read().strip().splitlines()[-1]); r=d['roofline']['kernels']
print('EARLY=$e', round(d['config']['ms_per_try'],3), 'head', round(r['k8_head_pair']['avg_launch_ms'],3), 'rk4', round(d['extra']['rk4']['ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
