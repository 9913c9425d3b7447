#!/usr/bin/env bash
# GPU-box helper: plain bench run, then the ncu launch list and one full
# capture of the named kernel (each ncu pass only after the plain run exits 0).
set -u
TAG=${1:-r1}
KREGEX=${2:-k_pc_accumulate}
ARGS="--steps 3 --warmup 3 --no-variants --no-cpu-baseline ${3:-}"
mkdir -p gpurun_out
timeout 600 python bench.py $ARGS > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py $ARGS > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s ${4:-4} -c ${5:-1} \
  -o gpurun_out/prof_$TAG python bench.py $ARGS > gpurun_out/ncu_full_$TAG.log 2>&1
echo done
