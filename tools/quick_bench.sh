#!/usr/bin/env bash
# quick bench lines (no variants / CPU baseline) for the given workloads
set -u
TAG=${1:-q}; shift || true
for w in "$@"; do
  timeout 600 python bench.py --workload $w --no-variants --no-cpu-baseline > gpurun_out/${TAG}_${w}.log 2>&1
  python - "$w" "gpurun_out/${TAG}_${w}.log" <<'PY'
import json, sys
w, path = sys.argv[1], sys.argv[2]
line = [l for l in open(path) if l.startswith("{")]
if not line:
    print(w, "FAILED"); print(open(path).read()[-1500:]); sys.exit(0)
d = json.loads(line[-1]); r = d.get("roofline") or {}
print(w, f"value={d['value']:.4g} ms={d['ms_per_step']:.4f} e2e={(d.get('e2e') or {}).get('value', 0):.4g}",
      "kernels", r.get("kernel_ms"), "frac", round(r.get("frac", 0), 3))
PY
done
