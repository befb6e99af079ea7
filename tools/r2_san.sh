#!/bin/bash
# compute-sanitizer over tools/sanitize_run.py: memcheck / synccheck / initcheck on everything;
# racecheck without the NCCL loopback sections and the CUDA-graph device loop (tool limits)
O=gpurun_out
rm -f $O/r2_san_summary.txt
for tool in memcheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python -u tools/sanitize_run.py > $O/r2_san_$tool.txt 2>&1
  echo "$tool rc=$? $(grep -c '^section' $O/r2_san_$tool.txt) sections; $(grep 'ERROR SUMMARY\|RACECHECK SUMMARY' $O/r2_san_$tool.txt)" >> $O/r2_san_summary.txt
done
SAN_NO_NCCL=1 SAN_NO_GRAPH=1 timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -u tools/sanitize_run.py > $O/r2_san_racecheck.txt 2>&1
echo "racecheck (no NCCL, no graph) rc=$? $(grep -c '^section' $O/r2_san_racecheck.txt) sections; $(grep 'RACECHECK SUMMARY' $O/r2_san_racecheck.txt)" >> $O/r2_san_summary.txt
