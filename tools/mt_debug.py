"""Debug: batched multi-target vs single-target fused on a threshold config."""
import sys
import numpy as np
import paper_1310_5541_b200 as pc
from paper_1310_5541_b200 import multitarget as mt

frac, scheme, cpp = float(sys.argv[1]), sys.argv[2], int(sys.argv[3])
n, T, K = 3000, 10, 8
frames, truth = mt.multi_target_scene(T, K, 160, seed=8)
centers = truth[:, 0].copy()
res = pc.ResampleConfig(frac, scheme)
grid = pc.BinGrid.pixel_aligned(160, 160, cpp)
mk = lambda c: pc.PcFilterConfig(n, pc.InitSpec(pc.StateVector(*c), "gauss", sigma=2.0),
                                 pc.DynamicsParams(0.5, 0.1, 1.0), res,
                                 pc.SpotLikelihood(pc.PsfParams(1.5, 10.0), pc.LikelihoodParams(10.0, 5)),
                                 grid=grid)
r = mt.multi_pcsir_track(frames, mk((0, 0, 0, 0, 20.0)), centers, 31)
for t in range(T):
    s = pc.pcsir_track([pc.ImageFrame(f) for f in frames], mk(centers[t]), pc.PhiloxRng(mt.target_seed(31, t)))
    g = pc.pcsir_track([pc.ImageFrame(f) for f in frames], mk(centers[t]), pc.PhiloxRng(mt.target_seed(31, t)), fused=False)
    d = np.abs(r.estimates[t] - s.estimates).max(axis=1)
    print(t, "res", r.resampled[t].astype(int), s.resampled.astype(int), "occ", r.occupied[t], "diff", d,
          "fused==general", np.array_equal(s.estimates, g.estimates), "ess", r.ess[t].round(1), s.ess.round(1))
