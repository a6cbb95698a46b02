#!/bin/bash
# Partial profiling round (run under gpurun from the repo root; 1 GPU): default bench lines
# and ncu launch lists for CONFIGS_BENCH, full captures of the dominant kernel for
# CONFIGS_FULL (gpurun copies back at most 64 MiB, so the full captures of all nine
# configurations do not fit in one call).
set -u
OUT=gpurun_out
mkdir -p $OUT
CONFIGS_BENCH=${CONFIGS_BENCH:-"1 2 3 4 5 6 7 8 9"}
CONFIGS_FULL=${CONFIGS_FULL:-"4 6 7 8"}
for c in $CONFIGS_BENCH; do
  timeout 600 python bench.py --config $c > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err || echo "bench cfg$c failed"
done
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
for c in $CONFIGS_BENCH; do
  [ "$c" = 1 ] && continue
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/launches_c$c.csv $CMD --config $c > $OUT/ncu_launch_c$c.log 2>&1
  echo "launches cfg$c rc=$?"
done
declare -A KREGEX=([2]="mci_row" [3]="mci_hilbert" [4]="mci_fsf_fb" [5]="mci_line" [6]="mci_anylen"
                   [7]="mci_anylen" [8]="mci_anylen" [9]="mci_avg_error_kernel")
declare -A SKIP=([2]=4 [3]=4 [4]=2 [5]=9 [6]=4 [7]=4 [8]=8 [9]=4)
for c in $CONFIGS_FULL; do
  timeout 900 ncu --set full --clock-control none --cache-control none --import-source on \
      -k regex:${KREGEX[$c]} -s ${SKIP[$c]} -c 1 -o $OUT/full_c$c $CMD --config $c > $OUT/ncu_full_c$c.log 2>&1
  echo "full cfg$c rc=$?"
done
