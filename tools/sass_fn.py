#!/usr/bin/env python
"""Print the SASS of one kernel (substring of its mangled name) from a .so:
usage: sass_fn.py LIB NAME_SUBSTR [--hist]"""
import collections
import re
import subprocess
import sys

lib, name = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
fns, cur = {}, None
for ln in out.splitlines():
    if "Function :" in ln:
        cur = ln.split("Function :")[1].strip()
        fns[cur] = []
    elif cur and re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+\S", ln):
        fns[cur].append(ln)
hit = [f for f in fns if name in f]
for f in hit:
    body = fns[f]
    print(f"== {f}: {len(body)} instructions")
    if "--hist" in sys.argv:
        c = collections.Counter(l.split("*/")[1].split()[0].split(".")[0].strip(";")
                                if not l.split("*/")[1].strip().startswith("@")
                                else l.split("*/")[1].split()[1].split(".")[0].strip(";")
                                for l in body)
        for k, v in c.most_common(40):
            print(f"{v:7d} {k}")
    else:
        print("\n".join(body))
