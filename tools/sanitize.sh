#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every kernel and variant
# (tools/sanitize_cases.py, reduced sizes).  Run under gpurun from the repo root (1 GPU);
# logs land in gpurun_out/sanitize/<tool>_<case>.log.  Usage: tools/sanitize.sh [case ...]
set -u
OUT=gpurun_out/sanitize
mkdir -p $OUT
CASES="${*:-row_kernel hilbert_kernel fused_kernel line_kernel fourstep anylen offgrid_complex_analysis sisr}"
SAN=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for c in $CASES; do
    extra=""
    [ $tool = memcheck ] && extra=""
    [ $tool = racecheck ] && extra="--racecheck-report all"
    timeout 900 $SAN --tool $tool $extra --error-exitcode 9 python tools/sanitize_cases.py $c \
        > $OUT/${tool}_$c.log 2>&1
    rc=$?
    echo "$tool $c rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $OUT/${tool}_$c.log | tail -1)"
  done
done
