set -u
mkdir -p gpurun_out
ARGS=${ARGS:-"--workload c5 --n 16777216 --steps 3 --warmup 3 --no-variants --no-cpu-baseline"}
timeout 600 python bench.py $ARGS > gpurun_out/c5s_plain.log 2>&1 || { echo plain failed; tail gpurun_out/c5s_plain.log; exit 1; }
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:${KRE:-k_sys_resample|k_pc_step1}" -s 6 -c 2 -o gpurun_out/prof_${TAG:-r1z} python bench.py $ARGS > gpurun_out/ncu_${TAG:-r1z}.log 2>&1
echo ncu_rc=$?
tail -3 gpurun_out/c5s_plain.log | cut -c1-400
