# ncu --set full of one k_mt_frame launch (c4 shape) after a plain run
set -u
mkdir -p gpurun_out
TAG=${1:-x}
ARGS="--workload c4 --steps 2 --warmup 3 --no-variants --no-cpu-baseline"
timeout 600 python bench.py $ARGS > gpurun_out/plain_${TAG}_c4.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k "regex:k_mt_frame" -s 4 -c 1 \
  -o gpurun_out/prof_${TAG}_c4 python bench.py $ARGS > gpurun_out/ncu_${TAG}_c4.log 2>&1
echo ncu_rc=$?
