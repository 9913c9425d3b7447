#!/usr/bin/env python
"""Print the key numbers of bench JSON lines (one per log file)."""
import json
import sys

for f in sys.argv[1:]:
    lines = [x for x in open(f) if x.startswith("{")]
    if not lines:
        print(f, "no JSON line")
        continue
    d = json.loads(lines[-1])
    r = d.get("roofline") or {}
    print(f"{d['config']['workload']}: {d['value']:.3e} {d['unit']}  {d['ms_per_step']:.4f} ms/step  "
          f"frac {r.get('frac', 0):.3f}  kernels {r.get('kernel_ms')}  e2e {d['e2e']['value']:.3e}")
    for k, v in (d.get("variants") or {}).items():
        print(f"   {k}: {v['value']:.3e} ({v['ms_per_step']:.4f} ms)")
