#!/usr/bin/env python
"""c2 pcSIR / SIR with the reference's default ResampleConfig() (ESS threshold
0.5, multinomial) through the fused loop, next to the benchmark setting
(threshold 1.0, systematic). Diagnostic only."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1310_5541_b200 as pc  # noqa: E402

wl = bench.WORKLOADS["c2"]
frames, truth = bench.frames_for(wl["width"], 43, wl["start"])
dev = torch.from_numpy(frames).cuda()
for label, res in (("systematic, threshold 1.0", pc.ResampleConfig(1.0, "systematic")),
                   ("default: multinomial, threshold 0.5", pc.ResampleConfig())):
    for method in ("pcSIR", "SIR"):
        def cfg():
            c, g = bench.make_cfg(pc, wl, 1.0 if method == "pcSIR" else None)
            kw = dict(n_particles=c.n_particles, init=c.init, dynamics=c.dynamics,
                      resampling=res, likelihood=c.likelihood)
            return (pc.PcFilterConfig(**kw, grid=g) if method == "pcSIR" else pc.FilterConfig(**kw))
        track = pc.pcsir_track if method == "pcSIR" else pc.sir_track
        track(dev[:3], cfg(), pc.PhiloxRng(1))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = track(dev[3:], cfg(), pc.PhiloxRng(1))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"{method:5s} {label:38s} path={r.path} {wl['n'] * 40 / dt:.3e} particle-updates/s "
              f"({dt / 40 * 1e3:.3f} ms/frame, resampled {int(np.sum(r.resampled))}/40, "
              f"rmse {np.sqrt(np.mean(np.sum((r.positions - truth[3:]) ** 2, axis=1))):.3f} px)")
