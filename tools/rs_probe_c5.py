#!/usr/bin/env python
"""c5-shape resampler phase split (CTA 0 globaltimer stamps of k_sys_resample:
pass 1, grid barrier, prefix, pass 2). usage: rs_probe_c5.py [N] [frames]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1310_5541_b200 as pc  # noqa: E402
from paper_1310_5541_b200 import _lib, synthesis  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 30
k = int(sys.argv[2]) if len(sys.argv) > 2 else 8
wl = dict(bench.WORKLOADS["c5"])
dev, _ = synthesis.spot_scene(k, 4096, wl["start"], seed=0)
cfg, grid = bench.make_cfg(pc, wl, 0.25, n)
c = bench.c_cfg(pc, _lib, cfg, grid, 1, use_graph=False)
st = _lib.stream()
_lib.check(_lib.lib().pcs_track_begin(_lib.ctx(), ctypes.byref(c), 4096, 4096, st))
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
    t2 = np.array(dbg[10:16], dtype=np.int64)
    print(f"frame {f} occ {int(occ[f])}: rs pass1 {(t2[1]-t2[0])/1e3:.1f} us, barrier "
          f"{(t2[2]-t2[1])/1e3:.1f}, prefix {(t2[3]-t2[2])/1e3:.1f}, pass2 {(t2[4]-t2[3])/1e3:.1f}, "
          f"cta0 total {(t2[4]-t2[0])/1e3:.1f}, last CTA end - cta0 start {(t2[5]-t2[0])/1e3:.1f}")
print(_lib.track_info())
