#!/bin/bash
# run under gpurun: bench config $CFG (default 2) with the default library and every exp/libmci_*.so named in
# $VARIANTS; TESTS="<pytest -k expr>" additionally runs those GPU tests against each variant
set -u
CFG=${CFG:-2}
OUT=gpurun_out; mkdir -p $OUT
B="python bench.py --config $CFG --no-cpu-baseline --no-e2e --steps ${STEPS:-40} --warmup 5"
show() { python - "$1" "$2" <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[2])); print(sys.argv[1], round(d["ms_per_step"], 4), "frac", round(d["roofline"]["frac"], 4))
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
}
$B > $OUT/abl_base.json 2> $OUT/abl_base.err; show base $OUT/abl_base.json
for v in ${VARIANTS:-}; do
  MCI_LIB=$PWD/exp/libmci_$v.so $B > $OUT/abl_$v.json 2> $OUT/abl_$v.err; show $v $OUT/abl_$v.json
  if [ -n "${TESTS:-}" ]; then
    MCI_LIB=$PWD/exp/libmci_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "$TESTS" > $OUT/abl_test_$v.log 2>&1
    echo "tests $v rc=$?"; tail -3 $OUT/abl_test_$v.log
  fi
done
$B > $OUT/abl_base2.json 2> $OUT/abl_base2.err; show base2 $OUT/abl_base2.json
