#!/bin/bash
# Warm-L2 per-stage DRAM bytes / durations of one DOPRI5 try (K8 head pair, K3 stages 4 + 5, K8 tail pair) under tuning knobs.
# usage: tools/tune.sh "<ENV=VAL ...>" tag
cd "$(dirname "$0")/.."
env $1 timeout 600 ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active -k "regex:gs_stage|gs_pair" -s 25 -c 4 --csv --log-file gpurun_out/tune_$2.csv python bench.py --steps 2 --warmup 3 --no-extra > gpurun_out/tune_$2.log 2>&1
