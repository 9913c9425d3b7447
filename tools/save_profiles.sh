#!/usr/bin/env bash
# Copy one round_profile.sh capture (gpurun_out/*_TAG*) into profiles/.
set -eu
TAG=$1
cp gpurun_out/launches_$TAG.csv profiles/${TAG}_launches.csv
python tools/ncu_summary.py gpurun_out/prof_$TAG.ncu-rep > profiles/${TAG}_ncu_summary.txt 2>&1
: > profiles/${TAG}_bench_lines.jsonl
for w in c1 c2 c3 c4 c5 ref; do
  grep "^{" gpurun_out/bench_${TAG}_$w.log | tail -1 >> profiles/${TAG}_bench_lines.jsonl || true
done
echo saved
