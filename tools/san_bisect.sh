#!/bin/bash
O=gpurun_out
for sec in base k3k6 r2 vector; do
  SAN_NO_NCCL=1 SAN_SECTIONS=$sec timeout 600 compute-sanitizer --tool racecheck --error-exitcode 9 python -X faulthandler -u tools/sanitize_run.py > $O/san_bis_$sec.txt 2>&1
  echo "$sec rc=$?" >> $O/san_bis_summary.txt
done
