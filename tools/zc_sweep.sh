# bench legs at several RKB_ZC settings ("yd,light,epart,heavy"); usage: tools/zc_sweep.sh TAG "legs" "set1 set2 ..."
TAG=$1; LEGS=$2; k=0
for zc in $3; do
  k=$((k+1))
  RKB_ZC=$zc timeout 600 python bench.py --legs $LEGS --steps 5 > gpurun_out/${TAG}_$k.log 2>&1
  echo "--- RKB_ZC=$zc"; python tools/legs_table.py gpurun_out/${TAG}_$k.log
done
