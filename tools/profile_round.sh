#!/bin/bash
# One pass of the round's profiling evidence (run under gpurun from the repo root):
#   bench line (all legs), ncu launch list, warm-L2 per-stage DRAM table, ncu --set full of one
#   DOPRI5 try and one RK4 step, dram bytes of one step of every other scheme leg.
#   Summaries are written on the box (tools/make_profiles.py) into gpurun_out/profiles_TAG/;
#   the bulky .ncu-rep files are deleted there except the DOPRI5 one (gpurun returns <= 64 MiB).
TAG=${1:-r2_v4}
O=gpurun_out
LEGS=adaptive,rk4,rk4_k3,repeats,try_loop,device_loop,halo,exposed,strong_emul,rk4_native,rk4_k6,midpoint_k6,midpoint_k3,exp512,small,e2e,cpu,cpu_full,euler,midpoint,modified_midpoint,cash_karp54,dopri5,rkf78,ab1,ab2,ab4,ab8,abm1,abm2,abm4,abm8
timeout 1200 python bench.py --legs $LEGS > $O/${TAG}_bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv \
    --log-file $O/${TAG}_launches.csv python bench.py --legs adaptive --steps 2 --warmup 3 > $O/${TAG}_launches.log 2>&1
bash tools/tune.sh "" ${TAG}
full() {  # leg, kernel regex, skip, count
  timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
      -k "regex:$2" -s $3 -c $4 -o $O/${TAG}_full_$1 -f \
      python bench.py --legs $1 --steps 2 --warmup 3 > $O/${TAG}_full_$1.log 2>&1
}
dram() {  # leg, kernel regex, skip, count: cold-L2 dram bytes per launch (csv)
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --kernel-name-base demangled -k "regex:$2" -s $3 -c $4 --csv \
      --log-file $O/${TAG}_dram_$1.csv python bench.py --legs $1 --steps 2 --warmup 3 > $O/${TAG}_dram_$1.log 2>&1
}
# one DOPRI5 try = the K8 head pair (stages 2 + 3), K3 stages 4 and 5, the K8 tail pair (6 + 7);
# skip the first try's k1 + 6 tries
full adaptive "gs_stage_kernel|gs_pair_kernel" 25 4
# RK4: K8 (2 pair launches per step, the default) and K3 (4 stage launches)
full rk4 "gs_pair_kernel" 6 2
full rk4_k3 "gs_stage_kernel" 12 4
dram euler "gs_stage_kernel" 3 1
dram midpoint "gs_pair_kernel" 3 1
dram midpoint_k3 "gs_stage_kernel" 6 2
dram modified_midpoint "gs_stage_kernel|gs_pair_kernel" 6 2
dram cash_karp54 "gs_stage_kernel" 18 6
dram dopri5 "gs_stage_kernel" 18 6
dram rkf78 "gs_stage_kernel" 39 13
for k in 1 2 4 8; do dram ab$k "gs_stage_kernel<.int.1$k," 2 1; done
for k in 1 2 4 8; do dram abm$k "gs_stage_kernel<.int.2$k," 2 1; done
python tools/make_profiles.py ${TAG} --out $O/profiles_${TAG} > $O/${TAG}_make.log 2>&1
rm -f $O/${TAG}_full_rk4.ncu-rep $O/${TAG}_full_rk4_k3.ncu-rep
du -sh $O
