#!/usr/bin/env python
"""c5 end-to-end breakdown (begin / upload / steps / end) of pcsir_track on
pinned host frames vs device frames. Diagnostic only (a single call also
pays the first device allocation of the frame buffer)."""
import ctypes, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import bench
import paper_1310_5541_b200 as pc
from paper_1310_5541_b200 import _lib
from paper_1310_5541_b200 import synthesis as syn
wl = bench.WORKLOADS["c5"]
dev, truth = syn.spot_scene(12, wl["width"], wl["start"], seed=0)
host = dev[2:12].cpu().pin_memory()
cfg, grid = bench.make_cfg(pc, wl, 0.25)
pc.pcsir_track(dev[:2], cfg, pc.PhiloxRng(1)); torch.cuda.synchronize()
def t(label, fn):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = fn(); torch.cuda.synchronize()
    print(f"{label:32s} {1e3*(time.perf_counter()-t0):9.2f} ms"); return r
cfg, grid = bench.make_cfg(pc, wl, 0.25)
t("whole pcsir_track (pinned)", lambda: pc.pcsir_track(host, cfg, pc.PhiloxRng(1)))
cfg, grid = bench.make_cfg(pc, wl, 0.25)
t("whole pcsir_track (device frames)", lambda: pc.pcsir_track(dev[2:12], cfg, pc.PhiloxRng(1)))
c = bench.c_cfg(pc, _lib, cfg, grid, 1, use_graph=True); st = _lib.stream()
t("pcs_track_begin", lambda: _lib.check(_lib.lib().pcs_track_begin(_lib.ctx(), ctypes.byref(c), 4096, 4096, st)))
d = t("H2D 10 frames", lambda: host.to("cuda", non_blocking=True))
K = 10
est = torch.empty((K, 5), dtype=torch.float64, device="cuda"); ess = torch.empty(K, dtype=torch.float64, device="cuda")
res = torch.empty(K, dtype=torch.uint8, device="cuda"); occ = torch.empty(K, dtype=torch.int64, device="cuda")
t("steps (10 frames)", lambda: _lib.check(_lib.lib().pcs_track_steps(_lib.ctx(), _lib.ptr(d), 0, K, _lib.ptr(est), _lib.ptr(ess), _lib.ptr(res), _lib.ptr(occ), st)))
out = _lib.PcsTrackResult()
t("end", lambda: _lib.lib().pcs_track_end(_lib.ctx(), ctypes.byref(out), st))
