"""Batched multi-target pcSIR (config 4): every target of one batched launch
equals a single-target fused pcsir_track with that target's RNG key, bit for
bit (estimates, ESS, resampling decisions, likelihood evaluations)."""

import numpy as np
import pytest

import paper_1310_5541_b200 as pc
from paper_1310_5541_b200 import multitarget as mt

pytestmark = pytest.mark.gpu


def _cfg(n, cpp=1):
    return pc.PcFilterConfig(
        n, pc.InitSpec(pc.StateVector(0, 0, 0, 0, 20.0), "gauss", sigma=2.0),
        pc.DynamicsParams(0.5, 0.1, 1.0), pc.ResampleConfig(1.0, "systematic"),
        pc.SpotLikelihood(pc.PsfParams(1.5, 10.0), pc.LikelihoodParams(10.0, 5)),
        grid=pc.BinGrid.pixel_aligned(160, 160, cpp))


@pytest.mark.parametrize("cpp,n", [(1, 3000), (2, 5000), (4, 4000)])   # cpp 4: many cells
                                                                    # outside the 24x24 window
def test_each_target_equals_single_target_filter(cuda, cpp, n):
    frames, truth = mt.multi_target_scene(12, 6, 160, seed=3)
    centers = truth[:, 0].copy()
    seed = 99
    r = mt.multi_pcsir_track(frames, _cfg(n, cpp), centers, seed)
    for t in range(12):
        cfg_t = pc.PcFilterConfig(
            n, pc.InitSpec(pc.StateVector(*centers[t]), "gauss", sigma=2.0),
            pc.DynamicsParams(0.5, 0.1, 1.0), pc.ResampleConfig(1.0, "systematic"),
            pc.SpotLikelihood(pc.PsfParams(1.5, 10.0), pc.LikelihoodParams(10.0, 5)),
            grid=pc.BinGrid.pixel_aligned(160, 160, cpp))
        single = pc.pcsir_track([pc.ImageFrame(f) for f in frames], cfg_t,
                                pc.PhiloxRng(mt.target_seed(seed, t)))
        assert single.path == "fused"
        assert np.array_equal(r.estimates[t], single.estimates), t
        assert np.array_equal(r.ess[t], single.ess), t
        assert np.array_equal(r.resampled[t], single.resampled), t
        assert int(r.likelihood_evals[t]) == single.likelihood_evals
    err = np.sqrt(np.mean(np.sum((r.estimates[:, :, :2] - truth[:, 1:, :2]) ** 2, axis=2)))
    assert err < 1.0


@pytest.mark.parametrize("frac,scheme,cpp", [(0.5, "systematic", 1), (0.2, "systematic", 4),
                                              (1.0, "multinomial", 2), (0.5, "multinomial", 1),
                                              (0.5, "multinomial", 4)])
def test_threshold_and_multinomial_equal_single_target(cuda, frac, scheme, cpp):
    """ResampleConfig other than (1.0, systematic) in the batched kernel: ESS-
    threshold frames that do not resample hand their weights to the next frame
    (log w = log w_prev + ll[cell], filtering.py:169-171, binning.py:190-192),
    and multinomial frames search the exact cdf (filtering.py:96-100). Every
    target still equals its single-target fused filter bit for bit."""
    n, T, K = 3000, 10, 8
    frames, truth = mt.multi_target_scene(T, K, 160, seed=8)
    centers = truth[:, 0].copy()
    res = pc.ResampleConfig(frac, scheme)
    lik = pc.SpotLikelihood(pc.PsfParams(1.5, 10.0), pc.LikelihoodParams(10.0, 5))
    grid = pc.BinGrid.pixel_aligned(160, 160, cpp)
    cfg = pc.PcFilterConfig(n, pc.InitSpec(pc.StateVector(0, 0, 0, 0, 20.0), "gauss", sigma=2.0),
                            pc.DynamicsParams(0.5, 0.1, 1.0), res, lik, grid=grid)
    r = mt.multi_pcsir_track(frames, cfg, centers, 31)
    if frac < 1.0:
        assert 0 < int(r.resampled.sum()) < T * K    # both kinds of frames occur
    for t in range(T):
        cfg_t = pc.PcFilterConfig(
            n, pc.InitSpec(pc.StateVector(*centers[t]), "gauss", sigma=2.0),
            pc.DynamicsParams(0.5, 0.1, 1.0), res,
            pc.SpotLikelihood(pc.PsfParams(1.5, 10.0), pc.LikelihoodParams(10.0, 5)), grid=grid)
        single = pc.pcsir_track([pc.ImageFrame(f) for f in frames], cfg_t,
                                pc.PhiloxRng(mt.target_seed(31, t)))
        assert single.path == "fused"
        assert np.array_equal(r.resampled[t], single.resampled), t
        assert np.array_equal(r.estimates[t], single.estimates), t
        assert np.array_equal(r.ess[t], single.ess), t
        assert int(r.likelihood_evals[t]) == single.likelihood_evals


def test_weighted_com_rejected(cuda):
    frames, truth = mt.multi_target_scene(1, 1, 160, seed=6)
    cfg = _cfg(1000)
    cfg = pc.PcFilterConfig(cfg.n_particles, cfg.init, cfg.dynamics, cfg.resampling, cfg.likelihood,
                            grid=cfg.grid, weighted_com=True)
    with pytest.raises(ValueError, match="unweighted centre"):
        mt.multi_pcsir_track(frames, cfg, truth[:, 0].copy(), 1)


def test_target_offset_selects_keys(cuda):
    frames, truth = mt.multi_target_scene(6, 3, 160, seed=4)
    centers = truth[:, 0].copy()
    full = mt.multi_pcsir_track(frames, _cfg(2000), centers, 5)
    half = mt.multi_pcsir_track(frames, _cfg(2000), centers[3:], 5, target_offset=3)
    assert np.array_equal(full.estimates[3:], half.estimates)


def test_many_tiles_per_target(cuda):
    # 200000 particles = 196 tiles per target (the digit accumulators are
    # not flushed inside a frame)
    frames, truth = mt.multi_target_scene(2, 3, 160, seed=5)
    centers = truth[:, 0].copy()
    n = 200_000
    r = mt.multi_pcsir_track(frames, _cfg(n), centers, 7)
    for t in range(2):
        cfg_t = pc.PcFilterConfig(
            n, pc.InitSpec(pc.StateVector(*centers[t]), "gauss", sigma=2.0),
            pc.DynamicsParams(0.5, 0.1, 1.0), pc.ResampleConfig(1.0, "systematic"),
            pc.SpotLikelihood(pc.PsfParams(1.5, 10.0), pc.LikelihoodParams(10.0, 5)),
            grid=pc.BinGrid.pixel_aligned(160, 160, 1))
        single = pc.pcsir_track([pc.ImageFrame(f) for f in frames], cfg_t,
                                pc.PhiloxRng(mt.target_seed(seed=7, t=t)))
        assert np.array_equal(r.estimates[t], single.estimates), t


def test_too_many_particles_per_target_rejected(cuda):
    frames, truth = mt.multi_target_scene(1, 1, 160, seed=6)
    with pytest.raises(Exception, match="too many particles per target"):
        mt.multi_pcsir_track(frames, _cfg(262_145), truth[:, 0].copy(), 1)


@pytest.mark.parametrize("cpp,sigma_pos", [(1, 1.2), (2, 1.5), (1, 2.0)])
def test_replicated_accumulators_with_outliers_equal_single_target(cuda, cpp, sigma_pos):
    """Phase A picks a 6/8/12-cell sub-window with 16/8/4 accumulator replicas
    from the previous frame's occupied span (pcs_multi.cuh). A large process
    noise makes the resampled (compact) cloud spread past that window every
    frame, so replicas and hashed outlier cells mix: the exact sums, hence
    every output, still equal the single-target fused filter bit for bit."""
    n, T, K = 4000, 6, 6
    frames, truth = mt.multi_target_scene(T, K, 160, seed=5)
    centers = truth[:, 0].copy()
    dyn = pc.DynamicsParams(sigma_pos, 0.1, 1.0)
    res = pc.ResampleConfig(1.0, "systematic")
    grid = pc.BinGrid.pixel_aligned(160, 160, cpp)

    def cfg(center):
        return pc.PcFilterConfig(
            n, pc.InitSpec(pc.StateVector(*center), "gauss", sigma=2.0), dyn, res,
            pc.SpotLikelihood(pc.PsfParams(1.5, 10.0), pc.LikelihoodParams(10.0, 5)), grid=grid)

    r = mt.multi_pcsir_track(frames, cfg((0, 0, 0, 0, 20.0)), centers, 17)
    # wider than the 6 / 8-cell windows a compact posterior selects
    assert int(r.occupied.max()) > (60 if cpp == 1 else 8)
    for t in range(T):
        single = pc.pcsir_track([pc.ImageFrame(f) for f in frames], cfg(centers[t]),
                                pc.PhiloxRng(mt.target_seed(17, t)))
        assert single.path == "fused"
        assert np.array_equal(r.estimates[t], single.estimates), t
        assert np.array_equal(r.ess[t], single.ess), t
        assert int(r.likelihood_evals[t]) == single.likelihood_evals
