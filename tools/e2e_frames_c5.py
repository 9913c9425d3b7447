#!/usr/bin/env python
"""c5: per-frame device time of the fused loop right after pcs_track_begin
(frame 0 starts from the wide initial cloud). Diagnostic only."""
import ctypes, os, sys
import torch
sys.path.insert(0, os.getcwd())
import bench
import paper_1310_5541_b200 as pc
from paper_1310_5541_b200 import _lib
from paper_1310_5541_b200 import synthesis as syn
wl = bench.WORKLOADS["c5"]
dev, truth = syn.spot_scene(12, wl["width"], wl["start"], seed=0)
cfg, grid = bench.make_cfg(pc, wl, 0.25)
pc.pcsir_track(dev[:2], cfg, pc.PhiloxRng(1)); torch.cuda.synchronize()
for use_graph in (1, 0):
    c = bench.c_cfg(pc, _lib, cfg, grid, 1, use_graph=use_graph); st = _lib.stream()
    _lib.check(_lib.lib().pcs_track_begin(_lib.ctx(), ctypes.byref(c), 4096, 4096, st))
    K = 10
    est = torch.empty((K, 5), dtype=torch.float64, device="cuda"); ess = torch.empty(K, dtype=torch.float64, device="cuda")
    res = torch.empty(K, dtype=torch.uint8, device="cuda"); occ = torch.empty(K, dtype=torch.int64, device="cuda")
    times = []
    for k in range(K):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(torch.cuda.current_stream())
        _lib.check(_lib.lib().pcs_track_steps(_lib.ctx(), _lib.ptr(dev[k:k + 1]), k, k + 1, _lib.ptr(est[k:]),
                                              _lib.ptr(ess[k:]), _lib.ptr(res[k:]), _lib.ptr(occ[k:]), st))
        e1.record(torch.cuda.current_stream())
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    info = _lib.track_info()
    print("graph" if use_graph else "plain", " ".join(f"{t:.2f}" for t in times), "occ", occ.tolist())
    print(info)
# per-kernel times of frames 0..2 (non-graph, CUDA events around each launch)
c = bench.c_cfg(pc, _lib, cfg, grid, 1, use_graph=0); st = _lib.stream()
_lib.check(_lib.lib().pcs_track_begin(_lib.ctx(), ctypes.byref(c), 4096, 4096, st))
for k in range(3):
    buf = (ctypes.c_double * 8)()
    _lib.check(_lib.lib().pcs_track_steps_timed(_lib.ctx(), _lib.ptr(dev[k:k + 1]), k, k + 1, _lib.ptr(est[k:]),
                                                _lib.ptr(ess[k:]), _lib.ptr(res[k:]), _lib.ptr(occ[k:]), buf, 8, st))
    torch.cuda.synchronize()
    print("frame", k, [round(buf[i], 3) for i in range(4)])
