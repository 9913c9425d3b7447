#!/usr/bin/env bash
# run tools/s1_probe.py with the PCS_S1_PROBE library variant, then restore
set -u
L=paper_1310_5541_b200/libpcsir_b200.so
cp $L /tmp/lib_orig.so
cp paper_1310_5541_b200/libpcsir_b200_s1probe.so $L
python tools/s1_probe.py "$@"
cp /tmp/lib_orig.so $L
