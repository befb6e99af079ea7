# configs[2] (64^3 RK4) under z-chunk settings; usage: tools/small_sweep.sh "settings"
for v in $1; do
  RKB_ZC=$v timeout 300 python bench.py --legs small --steps 5 > gpurun_out/sm_$v.log 2>&1
  echo "--- RKB_ZC=$v"; python tools/legs_table.py gpurun_out/sm_$v.log | grep gs64
done
