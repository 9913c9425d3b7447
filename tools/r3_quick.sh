# quick GPU check: full GPU tests, then c5 / c3 / c2 bench lines (no CPU baseline)
set -u
mkdir -p gpurun_out
TAG=${1:-q}
timeout 900 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider -x > gpurun_out/pytest_${TAG}.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_${TAG}.log
tail -4 gpurun_out/pytest_${TAG}.log
for w in c5 c3 c2; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --no-variants > gpurun_out/b_${TAG}_$w.log 2>&1
  python tools/show_bench.py gpurun_out/b_${TAG}_$w.log 2>/dev/null || grep "^{" gpurun_out/b_${TAG}_$w.log | cut -c1-400
done
