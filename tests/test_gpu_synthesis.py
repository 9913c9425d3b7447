"""GPU scene synthesis (synthesis.py:124-150): ideal frames against the
reference's render_clean_frame (golden) and the oracle's multi-spot
restatement; Poisson noise by its law (the numpy stream itself is not
reproducible on the device)."""

import numpy as np
import pytest
import scipy.stats

import paper_1310_5541_b200 as pc
from paper_1310_5541_b200 import synthesis as syn
from oracle import pcsir_oracle as orc
from conftest import golden

pytestmark = pytest.mark.gpu
PSF = pc.PsfParams(1.5, 10.0)


def _f32_close(got, want):
    # float64 fixed-point sum rounded once to float32: within one float32 ulp
    want32 = want.astype(np.float32)
    ulp = np.spacing(np.abs(want32)).astype(np.float64)
    assert np.all(np.abs(got.astype(np.float64) - want32.astype(np.float64)) <= ulp)


def test_clean_frame_matches_reference_golden(cuda):
    g = golden("synth")
    h, w = g["frames"].shape[1:]
    cfg = syn.SceneConfig(pc.PsfParams(float(g["sigma"]), float(g["bg"])), frames=1, width=w,
                          height=h)
    for s, f in zip(g["states"], g["frames"]):
        got = syn.render_clean_frame(s, cfg).cpu().numpy()
        _f32_close(got, f)


def test_multi_spot_ideal_matches_oracle_and_is_order_free(cuda):
    rng = np.random.default_rng(1)
    spots = np.stack([rng.uniform(-5, 133, 300), rng.uniform(-5, 101, 300),
                      rng.uniform(10, 40, 300)], axis=1)
    a = syn.render_frames(spots[None], 128, 96, PSF, noise=False)[0].cpu().numpy()
    b = syn.render_frames(spots[::-1][None].copy(), 128, 96, PSF, noise=False)[0].cpu().numpy()
    assert np.array_equal(a, b)
    want = orc.render_ideal(spots, 128, 96, 1.5, 10.0)
    np.testing.assert_allclose(a, want, rtol=2e-7, atol=1e-6)


@pytest.mark.parametrize("lam", [0.7, 4.0, 9.9, 10.0, 30.0, 150.0])
def test_poisson_noise_law(cuda, lam):
    f = syn.render_frames(np.zeros((1, 0, 3)), 512, 512, pc.PsfParams(1.5, lam), noise=True,
                          seed=7)[0].cpu().numpy().ravel()
    assert np.all(f == np.round(f)) and f.min() >= 0
    n = f.size
    assert abs(f.mean() - lam) < 5 * np.sqrt(lam / n)
    assert abs(f.var() - lam) < 6 * lam * np.sqrt(2.0 / n) + 6 * np.sqrt(lam / n)
    lo, hi = int(scipy.stats.poisson.ppf(1e-4, lam)), int(scipy.stats.poisson.ppf(1 - 1e-4, lam))
    ks = np.arange(lo, hi + 1)
    obs = np.array([np.sum(f == k) for k in ks], dtype=np.float64)
    exp = n * scipy.stats.poisson.pmf(ks, lam)
    keep = exp > 20
    obs, exp = obs[keep], exp[keep]
    exp *= obs.sum() / exp.sum()
    assert scipy.stats.chisquare(obs, exp).pvalue > 1e-4


def test_noise_is_deterministic_and_frame_indexed(cuda):
    spots = np.array([[[30.2, 20.7, 25.0]], [[31.0, 21.0, 25.0]]])
    a = syn.render_frames(spots, 64, 48, PSF, seed=3).cpu().numpy()
    b = syn.render_frames(spots, 64, 48, PSF, seed=3).cpu().numpy()
    c = syn.render_frames(spots, 64, 48, PSF, seed=4).cpu().numpy()
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    flat = syn.render_frames(np.zeros((2, 0, 3)), 256, 256, PSF, seed=5).cpu().numpy()
    r = np.corrcoef(flat[0].ravel(), flat[1].ravel())[0, 1]
    assert abs(r) < 0.01


def test_read_noise_adds_variance(cuda):
    f = syn.render_frames(np.zeros((1, 0, 3)), 512, 512, pc.PsfParams(1.5, 30.0), seed=9,
                          read_noise_std=2.0)[0].cpu().numpy().ravel()
    assert f.min() >= 0
    assert abs(f.mean() - 30.0) < 0.05
    assert abs(f.var() - 34.0) < 0.6


def test_scenes_track(cuda):
    frames, truth = syn.spot_scene(8, 64, (20.0, 32.0), seed=2)
    init = pc.InitSpec(pc.StateVector(20.0, 32.0, 0.5, 0.0, 20.0), "gauss", sigma=2.0)
    cfg = pc.PcFilterConfig(4000, init, pc.DynamicsParams(0.5, 0.1, 1.0),
                            pc.ResampleConfig(1.0, "systematic"),
                            pc.SpotLikelihood(PSF, pc.LikelihoodParams(10.0, 5)),
                            grid=pc.BinGrid.pixel_aligned(64, 64, 1))
    r = pc.pcsir_track([pc.ImageFrame(frames[k]) for k in range(8)], cfg, pc.PhiloxRng(1))
    rmse = np.sqrt(np.mean(np.sum((r.positions - truth) ** 2, axis=1)))
    assert rmse < 0.75
    mf, mt = syn.multi_target_scene_device(16, 3, 128, seed=1)
    assert mf.shape == (3, 128, 128) and mt.shape == (16, 4, 5)
