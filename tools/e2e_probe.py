#!/usr/bin/env python
"""Break the bench's e2e call (pcsir_track on host frames) into stages:
host stacking + pinning + H2D, pcs_track (begin / steps / end), results.
Diagnostic only."""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1310_5541_b200 as pc  # noqa: E402
from paper_1310_5541_b200 import _lib, filtering  # noqa: E402

wl_name = sys.argv[1] if len(sys.argv) > 1 else "c2"
wl = bench.WORKLOADS[wl_name]
K = int(sys.argv[2]) if len(sys.argv) > 2 else 100
frames_host, truth = bench.frames_for(wl["width"], K, wl["start"])
cfg, grid = bench.make_cfg(pc, wl, 1.0)
fr = [pc.ImageFrame(f) for f in frames_host]
pc.pcsir_track(fr[:5], cfg, pc.PhiloxRng(1))   # warm
torch.cuda.synchronize()


def t(label, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    print(f"{label:40s} {1e3 * (time.perf_counter() - t0):8.3f} ms")
    return r


for rep in range(2):
    cfg, grid = bench.make_cfg(pc, wl, 1.0)
    t("whole pcsir_track", lambda: pc.pcsir_track(fr, cfg, pc.PhiloxRng(1)))
    host = t("np.stack", lambda: np.stack([np.asarray(f.pixels, dtype=np.float32) for f in fr]))
    th = t("from_numpy + pin_memory", lambda: torch.from_numpy(host).pin_memory())
    dev = t("H2D", lambda: th.to("cuda", non_blocking=True))
    cfg, grid = bench.make_cfg(pc, wl, 1.0)
    c = bench.c_cfg(pc, _lib, cfg, grid, 1, use_graph=True)
    st = _lib.stream()
    t("pcs_track_begin", lambda: _lib.check(_lib.lib().pcs_track_begin(_lib.ctx(), ctypes.byref(c),
                                                                      wl["width"], wl["width"], st)))
    est = torch.empty((K, 5), dtype=torch.float64, device="cuda")
    ess = torch.empty(K, dtype=torch.float64, device="cuda")
    res = torch.empty(K, dtype=torch.uint8, device="cuda")
    occ = torch.empty(K, dtype=torch.int64, device="cuda")
    t("pcs_track_steps (first frame)", lambda: _lib.check(_lib.lib().pcs_track_steps(
        _lib.ctx(), _lib.ptr(dev), 0, 1, _lib.ptr(est), _lib.ptr(ess), _lib.ptr(res), _lib.ptr(occ), st)))
    t("pcs_track_steps (rest)", lambda: _lib.check(_lib.lib().pcs_track_steps(
        _lib.ctx(), _lib.ptr(dev), 1, K, _lib.ptr(est[1:]), _lib.ptr(ess[1:]), _lib.ptr(res[1:]),
        _lib.ptr(occ[1:]), st)))
    out = _lib.PcsTrackResult()
    t("pcs_track_end", lambda: _lib.check(_lib.lib().pcs_track_end(_lib.ctx(), ctypes.byref(out), st)))
    t("results to host", lambda: (est.cpu().numpy(), ess.cpu().numpy(), res.cpu().numpy()))
