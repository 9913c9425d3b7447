import cProfile, pstats, sys, os
sys.path.insert(0, os.getcwd())
import bench, torch
import paper_1310_5541_b200 as pc
wl = bench.WORKLOADS["c2"]
frames_host, truth = bench.frames_for(wl["width"], 100, wl["start"])
fr = [pc.ImageFrame(f) for f in frames_host]
cfg, grid = bench.make_cfg(pc, wl, 1.0)
pc.pcsir_track(fr[:5], cfg, pc.PhiloxRng(1)); torch.cuda.synchronize()
cfg, grid = bench.make_cfg(pc, wl, 1.0)
pr = cProfile.Profile(); pr.enable()
pc.pcsir_track(fr, cfg, pc.PhiloxRng(1)); torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
