#!/usr/bin/env python
"""Max |device log L - float64 oracle| of the likelihoods on config-3-like
inputs (states around the spot, I0 ~ N(20, 3)) and on uniform states."""
import sys
import pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_1310_5541_b200 as pc
from oracle import pcsir_oracle as orc
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1] / "tests"))
from conftest import spot_pixels  # noqa: E402

rng = np.random.default_rng(1)
W = 96
pix = rng.poisson(spot_pixels(40.3, 38.8, 20.0, 1.5, 10.0, W, W)).astype(np.float64)
n = 200_000
xs = (40.3 + rng.normal(0, 1.0, n)).astype(np.float32)
ys = (38.8 + rng.normal(0, 1.0, n)).astype(np.float32)
i0 = np.abs(rng.normal(20, 4, n)).astype(np.float32)
xs[:20000] = rng.uniform(-3, W + 3, 20000)
ys[:20000] = rng.uniform(-3, W + 3, 20000)
soa = torch.from_numpy(np.stack([xs, ys, np.zeros(n, np.float32), np.zeros(n, np.float32), i0])).cuda()
for sub, model in (("erf", 1), ("midpoint4", 2)):
    lik = pc.PoissonSpotLikelihood(pc.PsfParams(1.5, 10.0), pc.LikelihoodParams(10.0, 7), sub)
    ll = lik.loglik(soa, pc.ImageFrame(pix)).double().cpu().numpy()
    ref = orc.loglik_poisson(pix, xs, ys, i0, 1.5, 10.0, 7, model)
    err = np.abs(ll - ref)
    k = int(np.argmax(err))
    print(f"{sub}: max|d|={err.max():.3e} (ll={ref[k]:.3f}, x={xs[k]:.3f} y={ys[k]:.3f} "
          f"i0={i0[k]:.2f}) p99.9={np.quantile(err, 0.999):.2e} mean={err.mean():.2e} "
          f"max|ll|={np.abs(ref).max():.1f}")
lik = pc.SpotLikelihood(pc.PsfParams(1.5, 10.0), pc.LikelihoodParams(10.0, 5))
ll = lik.loglik(soa, pc.ImageFrame(pix)).double().cpu().numpy()
ref = orc.loglik_gauss(pix.astype(np.float32).astype(np.float64), xs.astype(np.float64),
                       ys.astype(np.float64), i0.astype(np.float64), 1.5, 10.0, 5, 10.0)
err = np.abs(ll - ref)
print(f"gauss: max|d|={err.max():.3e} mean={err.mean():.2e} max|ll|={np.abs(ref).max():.1f}")
