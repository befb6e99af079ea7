#!/bin/bash
# A/B of the paired opposite-direction z sweeps (RKB_ZPAIR) per stage kernel: ncu duration and
# DRAM bytes of every stage launch of one DOPRI5 try and one RK4 step (cold L2 per launch).
O=gpurun_out
for z in 1 0; do
  for leg in dopri5 rk4; do
    n=$([ $leg = dopri5 ] && echo 6 || echo 4)
    RKB_ZPAIR=$z timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --kernel-name-base demangled -k "regex:gs_stage_kernel" -s $((3*n)) -c $n --csv \
      --log-file $O/zab_${leg}_z$z.csv python bench.py --legs $leg --steps 2 --warmup 3 > $O/zab_${leg}_z$z.log 2>&1
  done
done
