import time, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, bench
import paper_1310_5541_b200 as pc
wl = bench.WORKLOADS["c2"]
frames, truth = bench.frames_for(wl["width"], 25, wl["start"])
dev = torch.from_numpy(frames).cuda()
for fused in (False, True):
    cfg, grid = bench.make_cfg(pc, wl, 1.0)
    pc.pcsir_track(dev[:3], cfg, pc.PhiloxRng(1), fused=fused)
    cfg, grid = bench.make_cfg(pc, wl, 1.0)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = pc.pcsir_track(dev[3:], cfg, pc.PhiloxRng(1), fused=fused)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(("fused" if fused else "general"), r.path, f"{wl['n'] * 22 / dt:.3e} particle-updates/s, {dt / 22 * 1e3:.3f} ms/frame")
