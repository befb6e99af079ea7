#!/bin/bash
# z-chunk length of the paired write-ahead class (2) at 512^3: ncu duration + DRAM bytes of the
# adaptive DOPRI5 write-ahead stage gs_stage_kernel<3,1,4> (2 launches each)
O=gpurun_out
for X in 16 24 32; do
  RKB_ZC="8,16,$X,48,4" timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --kernel-name-base demangled -k "regex:gs_stage_kernel<.int.3, .int.1, .int.4>" -s 2 -c 2 --csv \
    --log-file $O/zca_$X.csv python bench.py --legs adaptive --steps 1 --warmup 3 > $O/zca_$X.log 2>&1
done
for X in 16 32; do
  RKB_ZPAIR=0 RKB_ZC="8,16,$X,48,4" timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --kernel-name-base demangled -k "regex:gs_stage_kernel<.int.3, .int.1, .int.4>" -s 2 -c 2 --csv \
    --log-file $O/zca_np_$X.csv python bench.py --legs adaptive --steps 1 --warmup 3 > $O/zca_np_$X.log 2>&1
done
timeout 300 python bench.py --legs adaptive,rk4 --steps 5 --warmup 3 > $O/zca_bench.json 2>&1
