import numpy as np, torch, sys
sys.path.insert(0, '.')
import bench
import paper_1310_5541_b200 as pc
from paper_1310_5541_b200 import multitarget as mt, synthesis as syn
wl = bench.WORKLOADS["c4"]
T, K = 296, 15
dev, truth = syn.multi_target_scene_device(T, K, wl["width"], seed=0)
cfg, _ = bench.make_cfg(pc, wl, 1.0, n=100000, center=(0, 0, 0, 0, 20.0))
tr = mt.MultiTargetTracker(cfg, truth[:, 0], 1, K, wl["width"], wl["width"])
for k in range(K):
    tr.step(dev[k])
res = tr.results()
err = np.sqrt(np.sum((res.estimates[:, :, :2] - truth[:, 1:, :2]) ** 2, axis=2))  # (T, K)
print("median err per frame", np.round(np.median(err, axis=0), 3))
print("p90", np.round(np.percentile(err, 90, axis=0), 3))
print("max", np.round(err.max(axis=0), 2))
bad = np.where(err[:, -1] > 2)[0]
print("lost targets", len(bad), bad[:10])
for t in bad[:3]:
    print(t, "truth v", truth[t, 0, 2:4], "I0", truth[t, 0, 4], "est v", res.estimates[t, -1, 2:4], "err", np.round(err[t], 2))
# nearest-neighbour distance of lost targets
pos = truth[:, 1:, :2]
for t in bad[:3]:
    d = np.min(np.linalg.norm(pos[:, -1] - pos[t, -1], axis=1)[np.arange(T) != t])
    print("target", t, "nearest other spot at last frame", round(d, 2))
print("flags", np.count_nonzero(res.flags))
