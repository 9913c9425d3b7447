#!/usr/bin/env bash
# run tools/rs_probe_c5.py with the PCS_RS_PROBE library variant, then restore
set -u
L=paper_1310_5541_b200/libpcsir_b200.so
cp $L /tmp/lib_orig.so
cp paper_1310_5541_b200/libpcsir_b200_rsprobe.so $L
python tools/rs_probe_c5.py "$@"
cp /tmp/lib_orig.so $L
