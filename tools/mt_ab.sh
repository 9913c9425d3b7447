#!/usr/bin/env bash
# c4 A/B: bench line with the previous library (tools/old/) and the current one
set -u
cp paper_1310_5541_b200/libpcsir_b200.so /tmp/cur.so
# (build the previous library into tools/old/ first)
cp tools/old/libpcsir_b200_prev.so paper_1310_5541_b200/libpcsir_b200.so
bash tools/quick_bench.sh ${1}_prev c4
cp /tmp/cur.so paper_1310_5541_b200/libpcsir_b200.so
bash tools/quick_bench.sh ${1}_cur c4
