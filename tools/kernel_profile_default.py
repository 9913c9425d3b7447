#!/usr/bin/env python
"""Per-kernel times of a c2 frame with the reference's default resampling
(ESS threshold 0.5, multinomial) in the fused loop. Diagnostic only."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1310_5541_b200 as pc  # noqa: E402
from paper_1310_5541_b200 import _lib  # noqa: E402

wl = bench.WORKLOADS["c2"]
frames, _ = bench.frames_for(wl["width"], 30, wl["start"])
dev = torch.from_numpy(frames).cuda()
orig = bench.c_cfg


def c_cfg(*a, **k):
    c = orig(*a, **k)
    c.threshold_fraction = 0.5
    c.scheme = 1
    return c


bench.c_cfg = c_cfg
for cpp in (1.0, None):
    cfg, grid = bench.make_cfg(pc, wl, cpp)
    prof = bench.kernel_profile(torch, pc, _lib, cfg, grid, dev, 5, 20, 1, None)
    print("pcSIR" if cpp else "SIR", {k: round(v * 1e3, 1) for k, v in prof.items()}, "us")
