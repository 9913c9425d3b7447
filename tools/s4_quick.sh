# GPU-box helper: GPU tests, then c5 / c3 / c2 bench lines (kernel times). usage: bash tools/s4_quick.sh TAG [workloads...]
set -u
TAG=${1:-q}; shift || true
WL=${@:-c5 c3 c2}
mkdir -p gpurun_out
if [ -z "${SKIP_TESTS:-}" ]; then
timeout 900 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider -x > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/${TAG}_pytest.log
tail -3 gpurun_out/${TAG}_pytest.log
fi
LOGS=""
for w in $WL; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --no-variants > gpurun_out/${TAG}_$w.log 2>&1
  LOGS="$LOGS gpurun_out/${TAG}_$w.log"
done
python tools/show_bench.py $LOGS
