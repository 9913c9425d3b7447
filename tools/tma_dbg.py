import numpy as np, sys
sys.path.insert(0, '.')
import paper_1310_5541_b200 as pc
from paper_1310_5541_b200 import synthesis as syn
frames, truth = syn.spot_scene(4, 64, (20.0, 32.0), seed=2)
init = pc.InitSpec(pc.StateVector(20.0, 32.0, 0.5, 0.0, 20.0), "gauss", sigma=2.0)
cfg = pc.PcFilterConfig(2000, init, pc.DynamicsParams(0.5, 0.1, 1.0), pc.ResampleConfig(1.0, "systematic"),
                        pc.SpotLikelihood(pc.PsfParams(1.5, 10.0), pc.LikelihoodParams(10.0, 5)),
                        grid=pc.BinGrid.pixel_aligned(64, 64, 1))
r = pc.pcsir_track([pc.ImageFrame(frames[k]) for k in range(4)], cfg, pc.PhiloxRng(1))
print(r.path, r.positions)
