#!/usr/bin/env python
"""Per-phase cycle split of k_pc_step1 (CTA 0, clock64 at the phase barriers)
over a few frames of a c2/c5-like track. Diagnostic only.
usage: s1_probe.py WORKLOAD N CELL_PX [FRAMES]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1310_5541_b200 as pc  # noqa: E402
from paper_1310_5541_b200 import _lib  # noqa: E402

wl = bench.WORKLOADS[sys.argv[1]]
n = int(sys.argv[2])
cpp = 1.0 / float(sys.argv[3])
k = int(sys.argv[4]) if len(sys.argv) > 4 else 6
frames, _ = bench.frames_for(wl["width"], k, wl["start"])
dev = torch.from_numpy(frames).cuda()
cfg, grid = bench.make_cfg(pc, wl, cpp, n)
c = bench.c_cfg(pc, _lib, cfg, grid, 1, use_graph=False)
st = _lib.stream()
_lib.check(_lib.lib().pcs_track_begin(_lib.ctx(), ctypes.byref(c), wl["width"], wl["width"], st))
est = torch.empty((k, 5), dtype=torch.float64, device="cuda")
ess = torch.empty(k, dtype=torch.float64, device="cuda")
res = torch.empty(k, dtype=torch.uint8, device="cuda")
occ = torch.empty(k, dtype=torch.int64, device="cuda")
names = ["p1 (propagate/bin/rank)", "p2 (run offsets)", "p3 (scatter)", "p4 (run sums | gather)", "flush"]
for f in range(k):
    _lib.check(_lib.lib().pcs_track_steps(_lib.ctx(), _lib.ptr(dev[f:]), f, f + 1,
                                          _lib.ptr(est[f:]), _lib.ptr(ess[f:]),
                                          _lib.ptr(res[f:]), _lib.ptr(occ[f:]), st))
    torch.cuda.synchronize()
    dbg = (ctypes.c_int64 * 16)()
    _lib.check(_lib.lib().pcs_track_debug(_lib.ctx(), dbg, st))
    ph = np.array(dbg[10:15], dtype=np.float64)
    tot = float(dbg[15])
    print(f"frame {f} occ={int(occ[f])} total {tot / 1.965e3:.1f} us (CTA 0): " +
          ", ".join(f"{nm} {100 * v / tot:.1f}%" for nm, v in zip(names, ph)))
