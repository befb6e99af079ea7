# ncu --set full of single light-stage launches (euler, ab1, ab2, midpoint); run under gpurun
set -x
for pair in "euler:0:0:0" "ab1:11:0:0" "ab2:12:0:0" "midpoint:5:0:1"; do
  IFS=: read leg s a i <<< "$pair"
  timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:gs_stage_kernel<.int.$s, .int.$a, .int.$i>" --launch-skip 2 --launch-count 1 -o gpurun_out/prof_$leg -f \
    python bench.py --legs $leg --steps 2 --warmup 3 > gpurun_out/prof_$leg.log 2>&1
done
ls -la gpurun_out
