#!/bin/bash
# chunk-group size per stage class (RKB_ZPAIR="g0,g1,g2,g3,g4"): ncu duration + DRAM bytes of the
# stage launches of one fixed DOPRI5 step and one RK4 step at 512^3
O=gpurun_out
for G in "1,1,1,1,1" "1,2,2,1,1" "2,4,4,2,1" "4,8,8,4,1" "8,16,16,8,1"; do
  tag=$(echo $G | tr , _)
  for leg in dopri5 rk4; do
    n=$([ $leg = dopri5 ] && echo 6 || echo 4)
    RKB_ZPAIR=$G timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --kernel-name-base demangled -k "regex:gs_stage_kernel" -s $((3*n)) -c $n --csv \
      --log-file $O/zg_${leg}_$tag.csv python bench.py --legs $leg --steps 2 --warmup 3 > $O/zg_${leg}_$tag.log 2>&1
  done
done
