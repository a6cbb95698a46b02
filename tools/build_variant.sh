#!/bin/bash
# Build an experimental libmci variant: tools/build_variant.sh NAME "<extra nvcc flags>" [source ...]
# Recompiles the named csrc sources (default mci_row.cu) with the flags and links them with the
# objects of the regular build into exp/libmci_NAME.so (load with MCI_LIB=exp/libmci_NAME.so).
set -eu
NAME=$1; FLAGS=${2:-}; shift; shift || true
SRCS=${@:-mci_row.cu}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
PKG=$ROOT/paper_1802_10291_b200
mkdir -p $ROOT/exp/$NAME
OBJS=""
for o in $PKG/build/*.o; do
  b=$(basename $o .o); skip=0
  for s in $SRCS; do [ "$b" = "$s" ] && skip=1; done
  [ $skip = 0 ] && OBJS="$OBJS $o"
done
for s in $SRCS; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr -Xptxas -v $FLAGS -c -o $ROOT/exp/$NAME/$s.o $PKG/csrc/$s 2> $ROOT/exp/$NAME/$s.ptxas &
done
wait
for s in $SRCS; do OBJS="$OBJS $ROOT/exp/$NAME/$s.o"; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/exp/libmci_$NAME.so $OBJS
echo built exp/libmci_$NAME.so
