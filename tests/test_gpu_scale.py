"""Parity at the benchmark scale (BASELINE configs 3 and 5): the fused device
loop equals the independent step-by-step device path bit-for-bit, and the
fused frame's estimate equals the oracle's canonical sums on the fused path's
own states. At these sizes the code paths that small tests never reach run:
the step-1 per-cell digit flush (a cell's count in one CTA crossing
S1_CELL_FLUSH), several warp tiles per step-1 warp, the resampler's TMA ring past its first two buffers (>= 2 tiles per CTA), the
per-cell kernel over thousands of occupied cells (> 4096) and the SIR
likelihood's dynamic chunks — pcs_track_info reports which ran and the tests
assert it."""

import ctypes

import numpy as np
import pytest
import torch

import paper_1310_5541_b200 as pc
from oracle import pcsir_oracle as orc
from paper_1310_5541_b200 import _lib, binning, filtering, synthesis

pytestmark = pytest.mark.gpu

RES = pc.ResampleConfig(1.0, "systematic")
DYN = pc.DynamicsParams(0.5, 0.1, 1.0)


def _c5_cfg(n, start):
    init = pc.InitSpec(pc.StateVector(start[0], start[1], 0.5, 0.0, 20.0), "gauss", sigma=2.0)
    lik = pc.SpotLikelihood(pc.PsfParams(1.5, 10.0), pc.LikelihoodParams(10.0, 5))
    grid = pc.BinGrid(-0.5, -0.5, 0.25, 0.25, 16384, 16384)   # 4096 px at 0.25 px
    return pc.PcFilterConfig(n, init, DYN, RES, lik, grid=grid), grid


def _c3_cfg(n, start, cpp):
    init = pc.InitSpec(pc.StateVector(start[0], start[1], 0.5, 0.0, 20.0), "gauss", sigma=2.0)
    lik = pc.PoissonSpotLikelihood(pc.PsfParams(1.5, 10.0), pc.LikelihoodParams(10.0, 7), "erf")
    if cpp is None:
        return pc.FilterConfig(n, init, DYN, RES, lik), None
    cells = int(512 / cpp)
    grid = pc.BinGrid(-0.5, -0.5, cpp, cpp, cells, cells)
    return pc.PcFilterConfig(n, init, DYN, RES, lik, grid=grid), grid


def _track_states():
    """(5, N) float32 copy of the current fused track's states (after frame
    k-1 of a track stepped to k: the propagated, pre-resampling states)."""
    ctx, st = _lib.ctx(), _lib.stream()
    sp, ld = ctypes.c_void_p(), ctypes.c_int64()
    _lib.check(_lib.lib().pcs_track_states(ctx, ctypes.byref(sp), ctypes.byref(ld)))
    return sp.value, ld.value


def test_c5_shape_fused_equals_general_and_oracle(cuda):
    """Config 5's shape (4096^2 frames, 0.25 px cells on a 16384^2 grid) at
    N = 2^27: 296 step-1 CTAs, several warp tiles per warp (ticketed), 59
    resampler tiles per CTA, ~5k occupied cells at frame 0."""
    n = 1 << 27
    start = (2043.0, 2048.0)
    frames, truth = synthesis.spot_scene(3, 4096, start, seed=0)
    cfg, grid = _c5_cfg(n, start)
    a = pc.pcsir_track(frames, cfg, pc.PhiloxRng(7), fused=True)
    info = _lib.track_info()
    cfg2, _ = _c5_cfg(n, start)
    b = pc.pcsir_track(frames, cfg2, pc.PhiloxRng(7), fused=False)
    assert a.path == "fused" and b.path == "general"
    assert np.array_equal(a.estimates, b.estimates)
    assert np.array_equal(a.ess, b.ess)
    assert np.array_equal(a.resampled, b.resampled)
    assert a.likelihood_evals == b.likelihood_evals
    # the size-dependent paths ran
    assert info["s1_tiles_per_warp"] > 1, info
    assert info["rs_tiles_per_cta"] >= 2, info
    assert info["max_occupied"] > 4096, info        # (more than one CTA's worth of cells)
    assert np.sqrt(np.mean(np.sum((a.positions - truth) ** 2, axis=1))) < 0.5


def test_c5_shape_frame_estimate_equals_oracle(cuda):
    """Frame 0 of the fused loop at N = 2^27: cell ids, occupied count,
    dummies and the estimate / ESS equal the oracle's canonical results on
    the fused path's own propagated states (binning.py:97-112,157-172;
    filtering.py:112-114,88-90)."""
    n = 1 << 27
    start = (2043.0, 2048.0)
    frames, _ = synthesis.spot_scene(1, 4096, start, seed=0)
    cfg, grid = _c5_cfg(n, start)
    a = filtering.fused_track(frames, cfg, pc.PhiloxRng(11), method=1, grid=grid)
    ptr, ld = _track_states()
    soa = torch.empty((5, n), dtype=torch.float32, device="cuda")
    ident = torch.arange(n, dtype=torch.int32, device="cuda")
    buf = torch.empty((5, ld), dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib().pcs_gather(ptr, _lib.ptr(buf), ld, n, _lib.ptr(ident), _lib.stream()))
    soa.copy_(buf[:, :n])
    del buf, ident
    s32 = soa.cpu().numpy()
    gt = (grid.origin_x, grid.origin_y, grid.cell_width, grid.cell_height, grid.n_cols, grid.n_rows)
    ix, iy = orc.cell_indices(s32[0].astype(np.float64), s32[1].astype(np.float64), gt)
    flat = iy * gt[4] + ix
    unique, bin_of, counts = np.unique(flat, return_inverse=True, return_counts=True)
    assert int(a.likelihood_evals) == len(unique) > 4096
    # device partition of the same states (general path) is the oracle's
    part = binning.partition_device(soa, grid)
    assert np.array_equal(part.unique.cpu().numpy(), unique)
    assert np.array_equal(part.counts.cpu().numpy(), counts)
    d = binning.dummy_states_device(soa, grid, part, pc.DummyPlacement.CENTER_OF_MASS)
    dref = orc.dummies_exact(s32, bin_of.astype(np.int32), counts)
    assert np.array_equal(d.cpu().numpy(), dref)
    # weights from the oracle likelihood of the canonical dummies; the fused
    # frame's estimate / ESS are the canonical exact sums on those weights
    pix = frames[0].double().cpu().numpy()
    dd = dref.astype(np.float64)
    ll = orc.loglik_gauss(pix, dd[0], dd[1], dd[4], 1.5, 10.0, 5, 10.0)
    ll_dev = cfg.likelihood.loglik(d, pc.ImageFrame(pix), count=False).double().cpu().numpy()
    assert np.max(np.abs(ll_dev - ll)) < 1e-5
    logw = torch.from_numpy(ll_dev[bin_of]).cuda()
    w = filtering.normalize(pc.ParticleSet.from_device(soa, logw=logw)).w
    est, ess = orc.estimate_ess_exact(s32, w.cpu().numpy())
    assert np.array_equal(a.estimates[0], est)
    assert a.ess[0] == ess


def test_coarse_cells_per_cell_flush_fused_equals_general(cuda):
    """16 px cells at N = 2^24: every step-1 CTA adds tens of thousands of
    particles to the same few sub-window cells, so their digit accumulators
    are folded on the spot (count crossing S1_CELL_FLUSH, atomic-exchange
    flush) while other warps keep adding. Fused == general bit for bit."""
    n = 1 << 24
    start = (120.0, 128.0)
    frames, _ = synthesis.spot_scene(3, 256, start, seed=0)
    init = pc.InitSpec(pc.StateVector(start[0], start[1], 0.5, 0.0, 20.0), "gauss", sigma=2.0)
    lik = pc.SpotLikelihood(pc.PsfParams(1.5, 10.0), pc.LikelihoodParams(10.0, 5))
    grid = pc.BinGrid(-0.5, -0.5, 16.0, 16.0, 16, 16)
    mk = lambda: pc.PcFilterConfig(n, init, DYN, RES, lik, grid=grid)   # noqa: E731
    a = pc.pcsir_track(frames, mk(), pc.PhiloxRng(3), fused=True)
    info = _lib.track_info()
    b = pc.pcsir_track(frames, mk(), pc.PhiloxRng(3), fused=False)
    assert a.path == "fused" and b.path == "general"
    assert np.array_equal(a.estimates, b.estimates)
    assert np.array_equal(a.ess, b.ess)
    assert np.array_equal(a.resampled, b.resampled)
    assert info["s1_cell_flushes"] > 0, info


@pytest.mark.parametrize("cpp", [None, 0.5])
def test_c3_shape_fused_equals_general(cuda, cpp):
    """Config 3 (512^2, N = 1e7, erf-PSF Poisson 15x15): SIR runs the
    likelihood in dynamic chunks; pcSIR at 0.5 px. Fused == general."""
    n = 10_000_000
    start = (203.0, 256.0)
    frames, truth = synthesis.spot_scene(3, 512, start, seed=0)
    cfg, grid = _c3_cfg(n, start, cpp)
    track = pc.sir_track if cpp is None else pc.pcsir_track
    a = track(frames, cfg, pc.PhiloxRng(5), fused=True)
    info = _lib.track_info()
    cfg2, _ = _c3_cfg(n, start, cpp)
    b = track(frames, cfg2, pc.PhiloxRng(5), fused=False)
    assert a.path == "fused" and b.path == "general"
    assert np.array_equal(a.estimates, b.estimates)
    assert np.array_equal(a.ess, b.ess)
    assert np.array_equal(a.resampled, b.resampled)
    assert info["rs_tiles_per_cta"] >= 2, info
    if cpp is None:
        assert info["sir_chunk"] > 0, info
    assert np.sqrt(np.mean(np.sum((a.positions - truth) ** 2, axis=1))) < 0.5
