#!/bin/bash
# round-2 extra evidence: scheme sweep + K6 + halo legs (bench JSON), and compute-sanitizer on the
# sanitize workload (incl. the P2P allreduce, the graph loop and the unfused dataflow)
O=gpurun_out
timeout 900 python bench.py --legs halo,rk4_k6,midpoint_k6,euler,midpoint,modified_midpoint,cash_karp54,dopri5,rkf78,ab1,ab2,ab4,ab8,abm1,abm2,abm4,abm8 \
  --steps 10 --warmup 3 > $O/r2_schemes.json 2> $O/r2_schemes.err
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_run.py > $O/r2_san_$tool.txt 2>&1
  echo "$tool rc=$?" >> $O/r2_san_summary.txt
  tail -3 $O/r2_san_$tool.txt >> $O/r2_san_summary.txt
done
