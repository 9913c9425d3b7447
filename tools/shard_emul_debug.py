#!/usr/bin/env python
"""Debug: the emulated multi-rank sharded protocol step by step with a
synchronise after every call (CUDA_LAUNCH_BLOCKING=1 recommended)."""
import os, sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
import torch
from dataclasses import replace
import paper_1310_5541_b200 as pc
from paper_1310_5541_b200 import _lib, distributed as D

world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
rng = np.random.default_rng(7)
width, k_frames, n_global = 96, 4, 40000
xs = np.arange(width)
frames = []
x, y = 40.0, 45.0
for _ in range(k_frames):
    x += 0.5
    frames.append(rng.poisson(20.0 * np.outer(np.exp(-((xs - y) ** 2) / 4.5),
                                              np.exp(-((xs - x) ** 2) / 4.5)) + 10).astype(np.float32))
frames = torch.from_numpy(np.stack(frames)).cuda()
init = pc.InitSpec(pc.StateVector(40.0, 45.0, 0.5, 0.0, 20.0), "gauss", sigma=2.0)
cfg = pc.PcFilterConfig(n_global, init, pc.DynamicsParams(0.5, 0.1, 1.0),
                        pc.ResampleConfig(1.0, "systematic"),
                        pc.SpotLikelihood(pc.PsfParams(1.5, 10.0), pc.LikelihoodParams(10.0, 5)),
                        grid=pc.BinGrid.pixel_aligned(width, width, 1))
n = n_global // world
bcap = n // 4
ops = [D.DeviceShardOps(k_frames, _lib.new_ctx()) for _ in range(world)]

def sync(what):
    torch.cuda.synchronize()
    print("ok", what, flush=True)

for r, o in enumerate(ops):
    o.begin(replace(cfg, n_particles=n), width, width, r, world, n_global, 1 << 14, bcap, 77)
    sync(f"begin {r}")
for k in range(k_frames):
    boxes = []
    for r, o in enumerate(ops):
        boxes.append(o.step1(frames[k], k).clone()); sync(f"step1 k{k} r{r} box {boxes[-1].tolist()}")
    box = torch.stack(boxes).max(dim=0).values
    ls = []
    for r, o in enumerate(ops):
        ls.append(o.export(box).clone()); sync(f"export k{k} r{r}")
    limbs = torch.stack(ls).sum(dim=0)
    for r, o in enumerate(ops):
        o.import_bins(box, limbs); sync(f"import k{k} r{r}")
    tots = []
    for r, o in enumerate(ops):
        tots.append(o.total().clone()); sync(f"total k{k} r{r} {tots[-1].tolist()}")
    totals = torch.cat(tots)
    sends = []
    for r, o in enumerate(ops):
        sends.append(tuple(t.clone() for t in o.emit(totals))); sync(f"emit k{k} r{r}")
    for r, o in enumerate(ops):
        rp = sends[r - 1][1] if r > 0 else torch.zeros_like(sends[r][0])
        rn = sends[r + 1][0] if r < world - 1 else torch.zeros_like(sends[r][1])
        o.unpack(rp, rn); sync(f"unpack k{k} r{r}")
print([o.flags() for o in ops])
