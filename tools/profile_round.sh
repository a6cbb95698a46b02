#!/bin/bash
# Round profiling recipe (run under gpurun from the repo root; 1 GPU).
# Plain run first (must exit 0), then the ncu launch list of the same command,
# then one full capture of the dominant kernel per config.
set -u
OUT=gpurun_out
mkdir -p $OUT
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
for c in 2 3 4 5; do
  timeout 300 $CMD --config $c > $OUT/plain_c$c.log 2>&1 || { echo "plain run cfg$c failed"; continue; }
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/launches_c$c.csv $CMD --config $c > $OUT/ncu_launch_c$c.log 2>&1
  echo "launches cfg$c rc=$?"
done
declare -A KREGEX=([2]="mci_row" [3]="mci_hilbert" [4]="mci_fsf_fb" [5]="mci_line")
for c in 2 3 4 5; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX[$c]} -s 4 -c 1 \
      -o $OUT/full_c$c $CMD --config $c > $OUT/ncu_full_c$c.log 2>&1
  echo "full cfg$c rc=$?"
done
