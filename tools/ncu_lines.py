#!/usr/bin/env python
"""Join ncu per-SASS-instruction counts with nvdisasm line info:
instructions executed per CUDA source line for one kernel."""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, kregex, so = sys.argv[1], sys.argv[2], os.path.abspath(sys.argv[3])
# LAUNCH=k (env): the k-th captured launch of the kernel (1-based)
skip = ["--launch-skip", str(int(os.environ.get("LAUNCH", "1")) - 1)]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kregex}", *skip, "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ia, iex, ist = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index(
    "Warp Stall Sampling (All Samples)")
seen, data = set(), []
for r in rows[2:]:
    if len(r) <= iex or r[ia] in seen or not r[ia].startswith("0x"):
        continue
    seen.add(r[ia])
    data.append((int(r[ia], 16), float(r[iex] or 0), float(r[ist] or 0)))
base = min(a for a, _, _ in data)
# line info from the cubin
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True,
                     text=True).stdout
fn = None
line_of = {}
cur_line = None
in_fn = False
for ln in dis.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", ln)
    if m:
        in_fn = re.search(os.environ.get("SASS_RE", kregex), m.group(1)) is not None
        continue
    if not in_fn:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur_line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and cur_line:
        line_of[int(m.group(1), 16)] = cur_line
agg = collections.Counter()
st = collections.Counter()
for a, ex, s in data:
    l = line_of.get(a - base, "?")
    agg[l] += ex
    st[l] += s
tot = sum(agg.values())
print(f"total warp-instr {tot:.0f}")
for l, v in agg.most_common(int(os.environ.get("TOPN", "40"))):
    print(f"{v:12.0f} {100*v/tot:5.1f}%  stall_samples={st[l]:6.0f}  {l}")
