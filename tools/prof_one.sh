#!/bin/bash
# one full ncu capture under gpurun: tools/prof_one.sh <config> <kernel regex> <skip> <out name>
set -u
OUT=gpurun_out; mkdir -p $OUT
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --config $1"
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on -k regex:$2 -s $3 -c 1 -o $OUT/$4 $CMD > $OUT/ncu_$4.log 2>&1
echo "full rc=$?"; ls -la $OUT/$4.ncu-rep
