#!/usr/bin/env bash
# One GPU call: GPU tests + the default bench (c5) [+ extra bench args].
# usage (under gpurun): bash tools/gpu_round.sh TAG [extra bench.py args]
set -u
TAG=${1:-run}; shift || true
mkdir -p gpurun_out
if [ -z "${SKIP_TESTS:-}" ]; then
  timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -q -m gpu --timeout 900 -p no:cacheprovider ${PYTEST_ARGS:-} \
    > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/${TAG}_pytest.log
  tail -15 gpurun_out/${TAG}_pytest.log
fi
if [ -z "${SKIP_BENCH:-}" ]; then
  timeout 900 python bench.py "$@" > gpurun_out/${TAG}_bench.log 2>&1; echo bench_rc=$? >> gpurun_out/${TAG}_bench.log
  tail -c 4000 gpurun_out/${TAG}_bench.log
fi
