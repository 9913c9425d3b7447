#!/usr/bin/env python
"""Per source region: executed warp instructions and not-issued stall samples
by reason, from an ncu report (source page, SASS) joined with nvdisasm line
info of the matching .so.
usage: ncu_regions.py REP KREGEX SO UNITS file:lo-hi=name ..."""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, kregex, so, units = sys.argv[1], sys.argv[2], os.path.abspath(sys.argv[3]), float(sys.argv[4])
regions = []
for spec in sys.argv[5:]:
    fr, name = spec.split("=")
    f, rng = fr.split(":")
    lo, hi = (int(x) for x in rng.split("-"))
    regions.append((f, lo, hi, name))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kregex}", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ia, iex = hdr.index("Address"), hdr.index("Instructions Executed")
reasons = [h for h in hdr if h.startswith("stall_") and h.endswith("(Not Issued)")]
ir = [hdr.index(h) for h in reasons]
seen, data = set(), []
for r in rows[2:]:
    if len(r) <= iex or r[ia] in seen or not r[ia].startswith("0x"):
        continue
    seen.add(r[ia])
    data.append((int(r[ia], 16), float(r[iex] or 0), [float(r[i] or 0) for i in ir]))
base = min(a for a, _, _ in data)
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True,
                     text=True).stdout
line_of, cur, in_fn = {}, None, False
for ln in dis.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", ln)
    if m:
        in_fn = re.search(kregex, m.group(1)) is not None
        continue
    if not in_fn:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur
ins = collections.Counter()
st = collections.defaultdict(lambda: [0.0] * len(reasons))
for a, ex, s in data:
    f, l = line_of.get(a - base, ("?", 0))
    name = next((r[3] for r in regions if r[0] == f and r[1] <= l <= r[2]), f)
    ins[name] += ex
    for k, v in enumerate(s):
        st[name][k] += v
tot_i = sum(ins.values())
tot_s = sum(sum(v) for v in st.values()) or 1
short = [h[6:].replace(" (Not Issued)", "") for h in reasons]
print(f"total {tot_i / units:.2f} warp-instr/unit; stall samples {tot_s:.0f}")
for name, v in sorted(ins.items(), key=lambda kv: -sum(st[kv[0]])):
    s = st[name]
    top = sorted(zip(s, short), reverse=True)[:4]
    print(f"{v / units:6.2f}/unit {100 * sum(s) / tot_s:5.1f}% stalls  {name:14s} " +
          "  ".join(f"{n}={100 * x / tot_s:.1f}" for x, n in top if x > 0))
