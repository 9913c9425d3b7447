#!/usr/bin/env python
"""Per-kernel SASS instruction mix of a .so (static counts)."""
import collections
import re
import subprocess
import sys

so, pat = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
cur = None
mix = collections.defaultdict(collections.Counter)
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if m and cur:
        mix[cur][m.group(2)] += 1
for fn, c in mix.items():
    if pat and not re.search(pat, fn):
        continue
    print(f"== {fn[:90]}  total={sum(c.values())}")
    print("   " + ", ".join(f"{k}:{v}" for k, v in c.most_common(25)))
