#!/usr/bin/env python
"""Aggregate ncu_lines.py output (TOPN large) into named source regions.
usage: line_regions.py LINES_TXT N_UNITS file:lo-hi=name ..."""
import re
import sys
import collections

lines, units = sys.argv[1], float(sys.argv[2])
regions = []
for spec in sys.argv[3:]:
    fr, name = spec.split("=")
    f, rng = fr.split(":")
    lo, hi = (int(x) for x in rng.split("-"))
    regions.append((f, lo, hi, name))
agg = collections.Counter()
stall = collections.Counter()
tot = 0
for ln in open(lines):
    m = re.match(r"\s*(\d+)\s+[\d.]+%\s+stall_samples=\s*(\d+)\s+(\S+):(\d+)$", ln.rstrip())
    if not m:
        continue
    v, st, f, l = int(m.group(1)), int(m.group(2)), m.group(3), int(m.group(4))
    tot += v
    name = next((r[3] for r in regions if r[0] == f and r[1] <= l <= r[2]), f)
    agg[name] += v
    stall[name] += st
stot = sum(stall.values()) or 1
for k, v in agg.most_common():
    print(f"{v / units:7.2f} per unit  {100 * v / tot:5.1f}% instr  {100 * stall[k] / stot:5.1f}% stall samples  {k}")
