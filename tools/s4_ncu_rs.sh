# ncu --set full of k_sys_resample (steady-state frames) at the c5 shape (N = 2^24), after a plain run
set -u
mkdir -p gpurun_out
TAG=${1:-x}
SARGS="--workload c5 --n 16777216 --steps 3 --warmup 3 --no-variants --no-cpu-baseline"
timeout 600 python bench.py $SARGS > gpurun_out/plain_${TAG}_c5s.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k "regex:k_sys_resample" -s 3 -c 2 \
  -o gpurun_out/prof_${TAG}_rs python bench.py $SARGS > gpurun_out/ncu_${TAG}.log 2>&1
echo ncu_rc=$?
