#!/bin/bash
# Round profiling recipe (run under gpurun from the repo root; 1 GPU).
# 1. default bench line per config (cpu_baseline + e2e included), must exit 0;
# 2. ncu launch list (gpu__time_duration per launch) of the same command;
# 3. full captures of the dominant kernels listed in FULL (cache control off, so DRAM
#    bytes are those of the steady state, not of a flushed L2); gpurun copies back at most
#    64 MiB, so at most ~4 captures per call.
# Usage: [CONFIGS="1 2 ..."] [FULL="3 4 11"] tools/profile_round.sh <outdir under gpurun_out>
set -u
OUT=gpurun_out/${1:-r02}
mkdir -p $OUT
CONFIGS=${CONFIGS:-"1 2 3 4 5 6 7 8 9 10 11"}
FULL=${FULL:-""}
for c in $CONFIGS; do
  timeout 600 python bench.py --config $c > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err || echo "bench cfg$c failed"
done
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
for c in $CONFIGS; do
  [ "$c" = 1 ] && continue
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv \
      --log-file $OUT/launches_c$c.csv $CMD --config $c > $OUT/ncu_launch_c$c.log 2>&1
  echo "launches cfg$c rc=$?"
done
declare -A KREGEX=([2]="mci_row_kernel" [3]="mci_hilbert" [4]="mci_fsf_fb" [5]="mci_line" [6]="mci_anylen"
                   [7]="mci_anylen" [8]="mci_anylen" [9]="mci_avg_error_kernel" [10]="mci_rowg" [11]="mci_rowg")
declare -A SKIP=([2]=4 [3]=4 [4]=2 [5]=8 [6]=4 [7]=4 [8]=8 [9]=4 [10]=4 [11]=4)
declare -A COUNT=([5]=2)
for c in $FULL; do
  timeout 900 ncu --set full --clock-control none --cache-control none --import-source on \
      -k regex:${KREGEX[$c]} -s ${SKIP[$c]} -c ${COUNT[$c]:-1} -o $OUT/full_c$c $CMD --config $c > $OUT/ncu_full_c$c.log 2>&1
  echo "full cfg$c rc=$?"
done
