set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
SARGS="--workload c5 --n 16777216 --steps 3 --warmup 3 --no-variants --no-cpu-baseline"
timeout 600 python bench.py $SARGS > gpurun_out/plain_c5s.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k "regex:k_pc_step1|k_sys_resample" -s 6 -c 2 \
  -o gpurun_out/prof_r3a_c5s python bench.py $SARGS > gpurun_out/ncu_r3a.log 2>&1
echo ncu_rc=$?
grep "^{" gpurun_out/plain_c5s.log | cut -c1-300
