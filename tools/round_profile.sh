#!/usr/bin/env bash
# GPU-box helper: the default bench line (c2, with the CPU baseline), the other
# workloads, the reference arm, then the ncu launch list and full captures of
# the frame kernels (each ncu pass only after the plain run exited 0).
set -u
TAG=${1:-r1}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_${TAG}_c2.log 2>&1 || { echo "c2 bench failed"; exit 1; }
for w in c1 c3 c4 c5; do
  timeout 900 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_${TAG}_$w.log 2>&1
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_ref.log 2>&1
ARGS="--steps 3 --warmup 3 --no-variants --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py $ARGS > gpurun_out/ncu_launch_${TAG}.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k "regex:k_pc_step1|k_sys_resample|k_pc_bins" -s 6 -c 3 \
  -o gpurun_out/prof_${TAG} python bench.py $ARGS > gpurun_out/ncu_full_${TAG}.log 2>&1
echo done
