#!/bin/bash
# bench legs under a tuning env; prints one line per leg.  usage: tools/tune_legs.sh "<ENV>" legs tag
cd "$(dirname "$0")/.."
env $1 timeout 600 python bench.py --legs $2 --steps 5 > gpurun_out/tl_$3.log 2>&1
