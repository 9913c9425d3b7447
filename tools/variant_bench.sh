#!/usr/bin/env bash
# bench the same workload with several prebuilt library variants
# usage: variant_bench.sh TAG WORKLOAD lib_suffix...
set -u
TAG=$1; W=$2; shift 2
L=paper_1310_5541_b200/libpcsir_b200.so
cp $L /tmp/lib_orig.so
for v in "$@"; do
  cp paper_1310_5541_b200/libpcsir_b200_$v.so $L
  echo "== $v"; bash tools/quick_bench.sh ${TAG}_$v $W
done
cp /tmp/lib_orig.so $L
