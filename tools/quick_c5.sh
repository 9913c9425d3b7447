# GPU-box helper: GPU tests, then the c2 and c5 bench lines (kernel times)
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-variants > gpurun_out/b_c2.log 2>&1
timeout 600 python bench.py --workload c5 --no-cpu-baseline --no-variants > gpurun_out/b_c5.log 2>&1
python tools/show_bench.py gpurun_out/b_c2.log gpurun_out/b_c5.log
