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
tot = 0
for ln in open(lines):
    m = re.match(r"\s*(\d+)\s+[\d.]+%.*\s(\S+):(\d+)$", ln.rstrip())
    if not m:
        continue
    v, f, l = int(m.group(1)), m.group(2), int(m.group(3))
    tot += v
    name = next((r[3] for r in regions if r[0] == f and r[1] <= l <= r[2]), f)
    agg[name] += v
for k, v in agg.most_common():
    print(f"{v / units:7.2f} per unit  {100 * v / tot:5.1f}%  {k}")
