#!/usr/bin/env bash
# GPU-box helper (round 2): the default bench line (c5, with the CPU baseline
# and the likelihood roofline), the other workloads, the reference arm, then
# the ncu launch list of the default command and one full capture of the frame
# kernels at the c5 shape (N = 2^24; each ncu pass only after its plain run
# exited 0).
set -u
TAG=${1:-r2}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_${TAG}_c5.log 2>&1 || { echo "c5 bench failed"; tail gpurun_out/bench_${TAG}_c5.log; exit 1; }
for w in c1 c2 c3 c4; do
  timeout 900 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_${TAG}_$w.log 2>&1
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_ref.log 2>&1
ARGS="--steps 2 --warmup 3 --no-variants --no-cpu-baseline"
timeout 900 python bench.py $ARGS > gpurun_out/plain_${TAG}.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py $ARGS > gpurun_out/ncu_launch_${TAG}.log 2>&1
SARGS="--workload c5 --n 16777216 --steps 3 --warmup 3 --no-variants --no-cpu-baseline"
timeout 600 python bench.py $SARGS > gpurun_out/plain_${TAG}_c5s.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k "regex:k_pc_step1|k_sys_resample|k_pc_cells|k_pc_bins" -s 24 -c 4 \
  -o gpurun_out/prof_${TAG}_c5s python bench.py $SARGS > gpurun_out/ncu_full_${TAG}.log 2>&1
echo ncu_rc=$?
for w in c5 c1 c2 c3 c4 ref; do grep "^{" gpurun_out/bench_${TAG}_$w.log | tail -1 | cut -c1-300; done
