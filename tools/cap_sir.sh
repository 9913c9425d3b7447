#!/usr/bin/env bash
# ncu pipe utilisation of the SIR likelihood kernel at c3 (erf-Poisson) and c2 (Gaussian)
set -u
mkdir -p gpurun_out
for W in c3 c2; do
  ARGS="--workload $W --variant SIR --steps 3 --warmup 3 --no-variants --no-cpu-baseline"
  timeout 600 python bench.py $ARGS > gpurun_out/sir_${W}_plain.log 2>&1 || { echo plain failed; tail gpurun_out/sir_${W}_plain.log; exit 1; }
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_sir_propagate_lik -s 3 -c 1 -o gpurun_out/prof_${TAG:-r2}_sir_$W python bench.py $ARGS > gpurun_out/ncu_sir_$W.log 2>&1
  echo ncu_rc=$?
done
