#!/usr/bin/env bash
# like variant_bench.sh, with explicit bench.py arguments: TAG "ARGS" lib_suffix...
set -u
TAG=$1; ARGS=$2; shift 2
L=paper_1310_5541_b200/libpcsir_b200.so
cp $L /tmp/lib_orig.so
for v in "$@"; do
  cp paper_1310_5541_b200/libpcsir_b200_$v.so $L
  timeout 600 python bench.py $ARGS --no-variants --no-cpu-baseline > gpurun_out/${TAG}_$v.log 2>&1
  python - "$v" "gpurun_out/${TAG}_$v.log" <<'PY'
import json, sys
v, path = sys.argv[1], sys.argv[2]
line = [l for l in open(path) if l.startswith("{")]
if not line:
    print(v, "FAILED"); print(open(path).read()[-800:]); sys.exit(0)
d = json.loads(line[-1]); r = d.get("roofline") or {}
print(v, f"value={d['value']:.4g} ms={d['ms_per_step']:.4f}", "kernels", r.get("kernel_ms"))
PY
done
cp /tmp/lib_orig.so $L
