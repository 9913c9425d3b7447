#!/usr/bin/env python
"""Print the bins-kernel phase timestamps (globaltimer) of the last frame of a
short c2 pcSIR run. Diagnostic only."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1310_5541_b200 as pc  # noqa: E402
from paper_1310_5541_b200 import _lib  # noqa: E402

cpp = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
wl = bench.WORKLOADS["c2"]
frames, _ = bench.frames_for(wl["width"], 8, wl["start"])
dev = torch.from_numpy(frames).cuda()
n = int(sys.argv[2]) if len(sys.argv) > 2 else wl["n"]
cfg, grid = bench.make_cfg(pc, wl, cpp, n)
c = bench.c_cfg(pc, _lib, cfg, grid, 1, use_graph=False)
st = _lib.stream()
_lib.check(_lib.lib().pcs_track_begin(_lib.ctx(), ctypes.byref(c), 256, 256, st))
k = 8
est = torch.empty((k, 5), dtype=torch.float64, device="cuda")
ess = torch.empty(k, dtype=torch.float64, device="cuda")
res = torch.empty(k, dtype=torch.uint8, device="cuda")
occ = torch.empty(k, dtype=torch.int64, device="cuda")
for f in range(k):
    _lib.check(_lib.lib().pcs_track_steps(_lib.ctx(), _lib.ptr(dev[f:]), f, f + 1,
                                          _lib.ptr(est[f:]), _lib.ptr(ess[f:]),
                                          _lib.ptr(res[f:]), _lib.ptr(occ[f:]), st))
    torch.cuda.synchronize()
    dbg = (ctypes.c_int64 * 16)()
    _lib.check(_lib.lib().pcs_track_debug(_lib.ctx(), dbg, st))
    t = np.array(dbg[:8], dtype=np.int64)
    t2 = np.array(dbg[10:16], dtype=np.int64); print(f"frame {f} bins end->rs start {t2[0]-dbg[9]} ns; rs: pass1 {t2[1]-t2[0]}, barrier {t2[2]-t2[1]}, prefix {t2[3]-t2[2]}, pass2 {t2[4]-t2[3]}, cta0 total {t2[4]-t2[0]}, last CTA end - cta0 start {t2[5]-t2[0]}"); print("   bins phases", np.diff(t).tolist(),
          "entry->p0", t[0] - dbg[8], "p7->exit", dbg[9] - t[7])
