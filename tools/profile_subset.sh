set -u
OUT=gpurun_out
mkdir -p $OUT
for c in 2 3 5; do
  timeout 600 python bench.py --config $c > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err || echo "bench cfg$c failed"
done
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
for c in 2 5; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/launches_c$c.csv $CMD --config $c > $OUT/ncu_launch_c$c.log 2>&1
  echo "launches cfg$c rc=$?"
done
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on -k regex:mci_row -s 4 -c 1 -o $OUT/full_c2 $CMD --config 2 > $OUT/ncu_full_c2.log 2>&1; echo "full2 rc=$?"
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on -k regex:mci_line -s 8 -c 1 -o $OUT/full_c5 $CMD --config 5 > $OUT/ncu_full_c5.log 2>&1; echo "full5 rc=$?"
