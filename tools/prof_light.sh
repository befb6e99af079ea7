# ncu --set full of single stage launches; usage: tools/prof_light.sh TAG "leg:S:AD:I ..."
TAG=$1; shift
for pair in $@; do
  IFS=: read leg s a i <<< "$pair"
  timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:gs_stage_kernel<.int.$s, .int.$a, .int.$i>" --launch-skip 2 --launch-count 1 -o gpurun_out/${TAG}_$leg -f \
    python bench.py --legs ${leg%%-*} --steps 2 --warmup 3 > gpurun_out/${TAG}_$leg.log 2>&1
done
ls gpurun_out
