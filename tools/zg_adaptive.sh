#!/bin/bash
# chunk-group sizes on the adaptive DOPRI5 try (6 stage launches, ncu per launch, cold L2)
O=gpurun_out
for G in "1,2,2,1,1" "1,2,4,1,1" "1,4,4,1,1" "1,2,3,1,1"; do
  tag=$(echo $G | tr , _)
  RKB_ZPAIR=$G timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --kernel-name-base demangled -k "regex:gs_stage_kernel" -s 31 -c 6 --csv \
    --log-file $O/zga_$tag.csv python bench.py --legs adaptive --steps 1 --warmup 3 > $O/zga_$tag.log 2>&1
done
for G in "1,2,2,1,1" "1,2,4,1,1"; do
  tag=$(echo $G | tr , _)
  RKB_ZPAIR=$G timeout 300 python bench.py --legs adaptive --steps 5 --warmup 3 > $O/zga_bench_$tag.json 2>&1
done
