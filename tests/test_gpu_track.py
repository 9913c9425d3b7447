"""Filter steps and whole tracks on the device: golden steps from the
reference (replayed draws), fused device loop == general driver bit-for-bit,
pcSIR with sub-spacing cells == SIR bit-for-bit, oracle replay of the device's
own draws, driver semantics (degenerate frame index, point mass, no-resample)."""

import numpy as np
import pytest
import torch

import paper_1310_5541_b200 as pc
from conftest import assert_propagation_close, golden, spot_pixels
from oracle import pcsir_oracle as orc
from paper_1310_5541_b200 import rng as prng_mod
from paper_1310_5541_b200 import state

pytestmark = pytest.mark.gpu

W_RTOL = 1e-5
# The reference propagates in float64 and weights the UNROUNDED states; the
# device state is float32 (bit-exact to the canonical float32 form, within
# two float32 ulps of the reference's values). Position rounding
# (<= 1e-6 px) moves log L by up to ~|dlogL/dx| * 1e-6, i.e. a few 1e-5 for
# particles with large residuals — hence the looser tolerance when comparing
# with the reference's float64-state weights. Stage-wise (oracle on the
# device's own float32 states) the north-star 1e-5 holds.
W_RTOL_F64_STATES = 2e-4


def _oracle_weights(out_states32, prior, frame_pixels, lik_args, bin_map=None):
    """Reference weighting (imaging.py:137, filtering.py:69 / binning.py:189-192)
    on the device's float32 states; normalised (filtering.py:75-85)."""
    st = out_states32.astype(np.float64)
    if bin_map is None:
        ll = orc.loglik_gauss(frame_pixels, st[:, 0], st[:, 1], st[:, 4], *lik_args)
    else:
        d, bin_of = bin_map
        ll = orc.loglik_gauss(frame_pixels, d[0], d[1], d[4], *lik_args)[bin_of]
    lw = np.log(prior) + ll
    return orc.normalize(np.exp(lw - lw.max()))


def _check_states(dev_states, g, ref_states):
    """Propagated states: bit-exact against the canonical float32 form on the
    reference's replayed draws, within two float32 ulps of the reference."""
    s32, z32 = g["states"].T.astype(np.float32), g["normals"].T.astype(np.float32)
    dyn = (0.5, 0.1, 1.0, 1.0)
    assert np.array_equal(dev_states.T, orc.propagate_f32(s32, z32, *dyn))
    assert_propagation_close(np.ascontiguousarray(dev_states.T), ref_states.T, s32, z32, dyn)


# --- golden single steps (sis_step / pc_sis_step with the reference's draws) ----------
def test_sis_step_golden(cuda):
    g = golden("steps")
    frame = pc.ImageFrame(g["frame"])
    lik = pc.SpotLikelihood(pc.PsfParams(1.5, 10.0), pc.LikelihoodParams(10.0, 5))
    ps = pc.ParticleSet(g["states"], g["weights"])
    out = pc.sis_step(ps, frame, lik, pc.DynamicsParams(0.5, 0.1, 1.0),
                      prng_mod.ReplayNormals(g["normals"]))
    _check_states(out.states, g, g["sis_states"])
    w = pc.normalize(out).weights
    # stage-wise: oracle weighting of the device's float32 states
    want = _oracle_weights(out.states, g["weights"], g["frame"].astype(np.float32).astype(float),
                           (1.5, 10.0, 5, 10.0))
    np.testing.assert_allclose(w, want, rtol=W_RTOL, atol=1e-12)
    # against the reference's own float64-state weights
    np.testing.assert_allclose(w, orc.normalize(g["sis_weights"]), rtol=W_RTOL_F64_STATES,
                               atol=1e-12)


@pytest.mark.parametrize("cpp", [1, 2, 4])
def test_pc_sis_step_golden(cuda, cpp):
    g = golden("steps")
    frame = pc.ImageFrame(g["frame"])
    grid = pc.BinGrid.pixel_aligned(frame.width, frame.height, cpp)
    lik = pc.SpotLikelihood(pc.PsfParams(1.5, 10.0), pc.LikelihoodParams(10.0, 5))
    ps = pc.ParticleSet(g["states"], g["weights"])
    out, occ = pc.pc_sis_step(ps, frame, lik, pc.DynamicsParams(0.5, 0.1, 1.0), grid,
                              pc.DummyPlacement.CENTER_OF_MASS,
                              prng_mod.ReplayNormals(g["normals"]))
    assert occ == int(g[f"pc{cpp}_occ"])                 # bit-exact occupied-bin count
    assert lik.evals == int(g[f"pc{cpp}_evals"])
    _check_states(out.states, g, g[f"pc{cpp}_states"])
    w = pc.normalize(out).weights
    # stage-wise: canonical dummies of the device states, oracle likelihood per bin
    st32 = out.states.astype(np.float32)
    gt = (grid.origin_x, grid.origin_y, grid.cell_width, grid.cell_height, grid.n_cols,
          grid.n_rows)
    _, order, unique, starts, counts = orc.partition(st32.astype(np.float64), gt)
    bin_of = orc.bin_of_from_partition(len(st32), order, counts)
    d = orc.dummies_exact(np.ascontiguousarray(st32.T), bin_of, counts).astype(np.float64)
    want = _oracle_weights(st32, g["weights"], g["frame"].astype(np.float32).astype(float),
                           (1.5, 10.0, 5, 10.0), (d, bin_of))
    np.testing.assert_allclose(w, want, rtol=W_RTOL, atol=1e-12)
    np.testing.assert_allclose(w, orc.normalize(g[f"pc{cpp}_weights"]),
                               rtol=W_RTOL_F64_STATES, atol=1e-12)


def test_weight_ratios_identical_within_cells(cuda):
    # test_binning.py:146-162: broadcast of one likelihood per occupied cell
    rng = np.random.default_rng(4)
    frame = pc.ImageFrame(spot_pixels(20.0, 20.0, 22.0, 1.16, 10.0, 40, 40))
    st = np.zeros((200, 5))
    st[:, :2] = rng.uniform(15, 25, size=(200, 2))
    st[:, 4] = 22.0
    w0 = rng.uniform(0.1, 2.0, 200)
    ps = pc.ParticleSet(st, w0)
    grid = pc.BinGrid.pixel_aligned(40, 40, 1)
    lik = pc.SpotLikelihood(pc.PsfParams(1.16, 10.0), pc.LikelihoodParams(10.0, 4))
    out, occ = pc.pc_sis_step(ps, frame, lik, pc.DynamicsParams(0.0, 0.0, 0.0), grid,
                              pc.DummyPlacement.CENTER_OF_MASS, pc.PhiloxRng(0))
    assert lik.evals == occ
    occ_map = pc.assign_bins(out, grid)
    assert len(occ_map.members) == occ
    ratios = out.weights / ps.weights
    for idx in occ_map.members.values():
        np.testing.assert_allclose(ratios[idx], ratios[idx][0], rtol=1e-12)


# --- whole tracks ------------------------------------------------------------------------
def _c1_like(n=2000, k=12, seed=0, width=64):
    rng = np.random.default_rng(seed)
    frames, truth = [], []
    x, y = 20.0, 32.0
    for _ in range(k):
        x += 0.5
        truth.append((x, y))
        frames.append(pc.ImageFrame(rng.poisson(spot_pixels(x, y, 20.0, 1.5, 10.0, width, width))
                                    .astype(np.float64)))
    init = pc.InitSpec(pc.StateVector(20.0, 32.0, 0.5, 0.0, 20.0), "gauss", sigma=2.0)
    dyn = pc.DynamicsParams(0.5, 0.1, 1.0)
    return frames, np.array(truth), init, dyn


def _lik():
    return pc.SpotLikelihood(pc.PsfParams(1.5, 10.0), pc.LikelihoodParams(10.0, 5))


RES = pc.ResampleConfig(1.0, "systematic")


@pytest.mark.parametrize("cpp,placement", [(1, "com"), (4, "com"), (2, "coc"), (1, "coc")])
def test_fused_pcsir_equals_general(cuda, cpp, placement):
    frames, truth, init, dyn = _c1_like()
    pl = pc.DummyPlacement.CENTER_OF_MASS if placement == "com" else pc.DummyPlacement.CELL_CENTER
    cfg = pc.PcFilterConfig(2000, init, dyn, RES, _lik(),
                            grid=pc.BinGrid.pixel_aligned(64, 64, cpp), placement=pl)
    a = pc.pcsir_track(frames, cfg, pc.PhiloxRng(5), fused=True)
    cfg2 = pc.PcFilterConfig(2000, init, dyn, RES, _lik(),
                             grid=pc.BinGrid.pixel_aligned(64, 64, cpp), placement=pl)
    b = pc.pcsir_track(frames, cfg2, pc.PhiloxRng(5), fused=False)
    assert a.path == "fused" and b.path == "general"
    assert np.array_equal(a.estimates, b.estimates)
    assert np.array_equal(a.ess, b.ess)
    assert np.array_equal(a.resampled, b.resampled)
    assert a.likelihood_evals == b.likelihood_evals == cfg.likelihood.evals
    rmse = np.sqrt(np.mean(np.sum((a.positions - truth) ** 2, axis=1)))
    assert rmse < 0.75


@pytest.mark.parametrize("mult", [False, True])
def test_fused_pcsir_both_table_hashes(cuda, mult, monkeypatch):
    # the cell table's slot hash: the bit slice of (row, column) on grids with
    # 2^k columns, else (or with PCS_HT_MULT) the multiplicative hash with
    # linear probing. A wide cloud on fine cells puts many cells outside the
    # step-1 sub-window, so the first frame's queued form, the per-slot tables
    # and the resampler's lookups all go through it. Same results either way.
    if mult:
        monkeypatch.setenv("PCS_HT_MULT", "1")
    frames, truth, init, dyn = _c1_like(k=4)
    n = 60_000
    g = pc.BinGrid(-0.5, -0.5, 0.125, 0.125, 512, 512)   # 64 px / 0.125 px = 2^9 columns
    a = pc.pcsir_track(frames, pc.PcFilterConfig(n, init, dyn, RES, _lik(), grid=g),
                       pc.PhiloxRng(6), fused=True)
    b = pc.pcsir_track(frames, pc.PcFilterConfig(n, init, dyn, RES, _lik(), grid=g),
                       pc.PhiloxRng(6), fused=False)
    assert a.path == "fused" and b.path == "general"
    assert a.likelihood_evals > 4 * 1100     # more occupied cells than the 32 x 32 sub-window
    assert np.array_equal(a.estimates, b.estimates)
    assert np.array_equal(a.ess, b.ess)
    assert np.array_equal(a.resampled, b.resampled)
    assert a.likelihood_evals == b.likelihood_evals


def test_fused_sir_equals_general(cuda):
    frames, truth, init, dyn = _c1_like()
    a = pc.sir_track(frames, pc.FilterConfig(2000, init, dyn, RES, _lik()), pc.PhiloxRng(9),
                     fused=True)
    b = pc.sir_track(frames, pc.FilterConfig(2000, init, dyn, RES, _lik()), pc.PhiloxRng(9),
                     fused=False)
    assert a.path == "fused" and b.path == "general"
    assert np.array_equal(a.estimates, b.estimates)
    assert np.array_equal(a.ess, b.ess)
    assert a.likelihood_evals == 2000 * len(frames)


@pytest.mark.parametrize("method", ["sir", "pc"])
@pytest.mark.parametrize("small", [True, False])
def test_fused_resampling_many_tiles_heavy_weights(cuda, method, small, monkeypatch):
    # 2e5 particles -> 112 one-tile CTAs (k_sys_resample_small) or 53 CTAs of
    # the two-pass k_sys_resample (PCS_NO_RS_SMALL): grid barrier, exact CTA
    # prefixes; a sharp likelihood concentrates the weight so some tiles emit
    # more than one tile of slots (chunked emission)
    if not small:
        monkeypatch.setenv("PCS_NO_RS_SMALL", "1")
    frames, truth, init, dyn = _c1_like(k=5)
    n = 200_000
    sharp = pc.SpotLikelihood(pc.PsfParams(1.5, 10.0), pc.LikelihoodParams(1.5, 5))
    sharp2 = pc.SpotLikelihood(pc.PsfParams(1.5, 10.0), pc.LikelihoodParams(1.5, 5))
    if method == "sir":
        a = pc.sir_track(frames, pc.FilterConfig(n, init, dyn, RES, sharp), pc.PhiloxRng(3),
                         fused=True)
        b = pc.sir_track(frames, pc.FilterConfig(n, init, dyn, RES, sharp2), pc.PhiloxRng(3),
                         fused=False)
    else:
        g = pc.BinGrid.pixel_aligned(64, 64, 4)
        a = pc.pcsir_track(frames, pc.PcFilterConfig(n, init, dyn, RES, sharp, grid=g),
                           pc.PhiloxRng(3), fused=True)
        b = pc.pcsir_track(frames, pc.PcFilterConfig(n, init, dyn, RES, sharp2, grid=g),
                           pc.PhiloxRng(3), fused=False)
    assert a.path == "fused" and b.path == "general"
    assert np.min(a.ess) < n / 50   # concentrated: some tiles carry many slots
    assert np.array_equal(a.estimates, b.estimates)
    assert np.array_equal(a.ess, b.ess)
    assert np.array_equal(a.resampled, b.resampled)


@pytest.mark.parametrize("frac", [0.2, 0.5])
def test_fused_sir_threshold_resampling_equals_general(cuda, frac):
    # ESS-threshold resampling on the device (filtering.py:169-170): frames
    # that do not resample carry their normalised weights into the next
    # update (log w = log w_prev + ll) without a host round trip
    frames, truth, init, dyn = _c1_like(n=3000, k=12)
    res = pc.ResampleConfig(frac, "systematic")
    a = pc.sir_track(frames, pc.FilterConfig(3000, init, dyn, res, _lik()), pc.PhiloxRng(4))
    b = pc.sir_track(frames, pc.FilterConfig(3000, init, dyn, res, _lik()), pc.PhiloxRng(4),
                     fused=False)
    assert a.path == "fused" and b.path == "general"
    assert 0 < int(np.sum(a.resampled)) < len(frames)   # both kinds of frames occur
    assert np.array_equal(a.resampled, b.resampled)
    assert np.array_equal(a.estimates, b.estimates)
    assert np.array_equal(a.ess, b.ess)


@pytest.mark.parametrize("frac,cpp", [(0.2, 1), (0.5, 1), (0.5, 4)])
def test_fused_pcsir_threshold_resampling_equals_general(cuda, frac, cpp):
    # ESS-threshold resampling in the fused pcSIR loop: frames after a
    # non-resampling frame carry per-particle prior weights (log w = log w_prev +
    # ll[cell], binning.py:190-192) and finish per particle on the device
    frames, truth, init, dyn = _c1_like(n=3000, k=12)
    res = pc.ResampleConfig(frac, "systematic")
    g = pc.BinGrid.pixel_aligned(64, 64, cpp)
    a = pc.pcsir_track(frames, pc.PcFilterConfig(3000, init, dyn, res, _lik(), grid=g),
                       pc.PhiloxRng(4))
    lik_b = _lik()
    b = pc.pcsir_track(frames, pc.PcFilterConfig(3000, init, dyn, res, lik_b, grid=g),
                       pc.PhiloxRng(4), fused=False)
    assert a.path == "fused" and b.path == "general"
    assert 0 < int(np.sum(a.resampled)) < len(frames)   # both kinds of frames occur
    assert np.array_equal(a.resampled, b.resampled)
    assert np.array_equal(a.estimates, b.estimates)
    assert np.array_equal(a.ess, b.ess)
    assert a.likelihood_evals == b.likelihood_evals == lik_b.evals


def _rounding_edge_positions(cpp, ncols):
    """Cell edges b and the float32 positions just below them whose float32
    p - origin rounds ONTO the edge (a float32 cell estimate that trusted
    them would put them in b's cell; binning.py:61-67 puts them below)."""
    out, n_bad = [], 0
    for k in range(1, ncols):
        b = np.float32(-0.5 + k / cpp)
        below = []
        p = b
        for _ in range(6):
            p = np.nextafter(p, np.float32(-np.inf))
            t32 = np.float32(np.float32(p + np.float32(0.5)) * np.float32(cpp))
            if np.floor(t32) != np.floor((float(p) + 0.5) * cpp):
                below.append(p)
        if below:
            out += [b] + below
            n_bad += len(below)
    assert n_bad > 0
    return np.array(out, dtype=np.float32)


@pytest.mark.parametrize("cpp", [1, 2, 4])
def test_fused_step_cell_edges_exact(cuda, cpp):
    """binning.py:61-67 cell_indices on positions at and just below cell edges:
    the fused step's occupied-cell count equals the float64 count."""
    from paper_1310_5541_b200 import _lib
    import ctypes
    xs = _rounding_edge_positions(cpp, 16 * cpp)
    n = 2 * len(xs)
    st = np.zeros((n, 5), dtype=np.float32)
    st[:, 4] = 20.0
    st[: len(xs), 0], st[: len(xs), 1] = xs, np.float32(7.3)     # edges along x
    st[len(xs):, 0], st[len(xs):, 1] = np.float32(7.3), xs       # edges along y
    grid = pc.BinGrid.pixel_aligned(16, 16, cpp)
    want = len({(int(np.floor((float(x) + 0.5) * cpp)), int(np.floor((float(y) + 0.5) * cpp)))
                for x, y in st[:, :2]})
    c = _lib.PcsTrackCfg()
    c.method, c.placement, c.n_particles = 1, 0, n
    c.init = pc.InitSpec(pc.StateVector(8, 8, 0, 0, 20.0), "point").to_c()
    c.dyn = pc.DynamicsParams(0.0, 0.0, 0.0).to_c()   # states stay exactly as written
    c.spot = _lik().spot_c()
    c.grid = grid.to_c()
    c.seed, c.frame0, c.use_graph, c.threshold_fraction = 3, 0, 0, 1.0
    frame = torch.full((1, 16, 16), 10.0, dtype=torch.float32, device="cuda")
    ctx, stream = _lib.ctx(), _lib.stream()
    _lib.check(_lib.lib().pcs_track_begin(ctx, ctypes.byref(c), 16, 16, stream))
    sp, ld = ctypes.c_void_p(), ctypes.c_int64()
    _lib.check(_lib.lib().pcs_track_states(ctx, ctypes.byref(sp), ctypes.byref(ld)))
    buf = torch.zeros((5, ld.value), dtype=torch.float32, device="cuda")
    buf[:, :n] = torch.from_numpy(np.ascontiguousarray(st.T)).cuda()
    ident = torch.arange(n, dtype=torch.int32, device="cuda")
    # overwrite the initial cloud with the crafted states (SoA, stride ld)
    _lib.check(_lib.lib().pcs_gather(_lib.ptr(buf), sp.value, ld.value, n, _lib.ptr(ident), stream))
    est = torch.empty((1, 5), dtype=torch.float64, device="cuda")
    ess = torch.empty(1, dtype=torch.float64, device="cuda")
    res = torch.empty(1, dtype=torch.uint8, device="cuda")
    occ = torch.empty(1, dtype=torch.int64, device="cuda")
    _lib.check(_lib.lib().pcs_track_steps(ctx, _lib.ptr(frame), 0, 1, _lib.ptr(est), _lib.ptr(ess),
                                          _lib.ptr(res), _lib.ptr(occ), stream))
    out = _lib.PcsTrackResult()
    _lib.check(_lib.lib().pcs_track_end(ctx, ctypes.byref(out), stream))
    torch.cuda.synchronize()
    assert int(occ[0]) == want


def test_pcsir_tiny_cells_bitidentical_to_sir(cuda):
    # SPEC acceptance #1 / test_binning.py:208-226: 1e-5 px cells (64-bit keys)
    frames, truth, init, dyn = _c1_like(n=500, k=10)
    init = pc.InitSpec(pc.StateVector(20.0, 32.0, 0.5, 0.0, 20.0), "point")
    sir = pc.sir_track(frames, pc.FilterConfig(500, init, dyn, RES, _lik()), pc.PhiloxRng(11))
    tiny = pc.BinGrid(-0.5, -0.5, 1e-5, 1e-5, 64 * 10 ** 5, 64 * 10 ** 5)
    pcr = pc.pcsir_track(frames, pc.PcFilterConfig(500, init, dyn, RES, _lik(), grid=tiny),
                         pc.PhiloxRng(11))
    assert np.array_equal(sir.estimates, pcr.estimates)
    assert np.array_equal(sir.ess, pcr.ess)
    assert np.array_equal(sir.resampled, pcr.resampled)


def test_track_replays_into_oracle(cuda):
    """The oracle's restatement of the reference driver, fed the device's own
    draws, reproduces the device estimates (first frames before any
    rounding-induced divergence) within 1e-5 and the same RMSE regime."""
    frames, truth, init, dyn = _c1_like(n=3000, k=8)
    seed = 21
    r = pc.pcsir_track(frames, pc.PcFilterConfig(3000, init, dyn, RES, _lik(),
                                                 grid=pc.BinGrid.pixel_aligned(64, 64, 1)),
                       pc.PhiloxRng(seed))

    def dev_normals(f, n):
        return state.device_normals(seed, f, n).double().cpu().numpy()

    def dev_init(n):
        z = torch.empty((2, n), dtype=torch.float32, device="cuda")
        from paper_1310_5541_b200 import _lib
        _lib.check(_lib.lib().pcs_philox_init_normals(seed, 0, n, _lib.ptr(z), n, _lib.stream()))
        return z.double().cpu().numpy()

    replay = orc.PhiloxReplay(seed, normals_fn=dev_normals, init_fn=dev_init)
    lik = orc.SpotModel(1.5, 10.0, 10.0, 5)
    est, ess, res, evals = orc.track([f.pixels for f in frames], 3000,
                                     [20.0, 32.0, 0.5, 0.0, 20.0], 2.0, [0.5, 0.5, 0.1, 0.1, 1.0],
                                     1.0, lik, replay, grid=(-0.5, -0.5, 1.0, 1.0, 64, 64))
    np.testing.assert_allclose(r.estimates[0], est[0], rtol=W_RTOL)
    assert r.ess[0] == pytest.approx(ess[0], rel=W_RTOL)
    rm_dev = np.sqrt(np.mean(np.sum((r.positions - truth) ** 2, axis=1)))
    rm_orc = np.sqrt(np.mean(np.sum((est[:, :2] - truth) ** 2, axis=1)))
    assert abs(rm_dev - rm_orc) < 0.1


def test_point_mass_single_frame_exact(cuda):
    truth = pc.StateVector(20.0, 24.0, 0.0, 0.0, 22.0)
    frame = pc.ImageFrame(spot_pixels(20.0, 24.0, 22.0, 1.16, 10.0, 48, 48))
    lik = pc.SpotLikelihood(pc.PsfParams(1.16, 10.0), pc.LikelihoodParams(10.0, 4))
    cfg = pc.FilterConfig(16, pc.InitSpec(truth, "point"), pc.DynamicsParams(0.0, 0.0, 0.0),
                          likelihood=lik)
    result = pc.sir_track([frame], cfg, pc.PhiloxRng(0))
    assert np.array_equal(result.estimates[0], truth.as_array())


class ConstantLikelihood:
    def __init__(self, value):
        self.value = value

    def batch(self, states, frame):
        return np.full(states.shape[0], self.value)


def test_constant_likelihood_never_resamples(cuda):
    frames = [pc.ImageFrame(np.zeros((8, 8)))] * 12
    init = pc.InitSpec(pc.StateVector(4, 4, 0, 0, 1.0), "uniform", width=2.0)
    cfg = pc.FilterConfig(64, init, pc.DynamicsParams(0.1, 0.1, 0.0),
                          pc.ResampleConfig(threshold_fraction=0.99),
                          likelihood=ConstantLikelihood(0.5))
    result = pc.sir_track(frames, cfg, pc.PhiloxRng(3))
    assert not result.resampled.any()
    np.testing.assert_allclose(result.ess, 64.0, rtol=1e-6)


def test_degenerate_error_carries_frame_index(cuda):
    class DiesOnThird(ConstantLikelihood):
        def __init__(self):
            super().__init__(1.0)
            self.calls = 0

        def batch(self, states, frame):
            self.calls += 1
            if self.calls == 3:
                return np.zeros(states.shape[0])
            return super().batch(states, frame)

    frames = [pc.ImageFrame(np.zeros((8, 8)))] * 3
    cfg = pc.FilterConfig(8, pc.InitSpec(pc.StateVector(4, 4, 0, 0, 1)),
                          pc.DynamicsParams(0.0, 0.0, 0.0), likelihood=DiesOnThird())
    with pytest.raises(pc.DegenerateWeightsError) as err:
        pc.sir_track(frames, cfg, pc.PhiloxRng(0))
    assert err.value.frame_index == 2


def test_tracking_is_deterministic(cuda):
    frames, truth, init, dyn = _c1_like(n=4000, k=6)
    cfg = lambda: pc.PcFilterConfig(4000, init, dyn, RES, _lik(),  # noqa: E731
                                    grid=pc.BinGrid.pixel_aligned(64, 64, 4))
    a = pc.pcsir_track(frames, cfg(), pc.PhiloxRng(42))
    b = pc.pcsir_track(frames, cfg(), pc.PhiloxRng(42))
    assert np.array_equal(a.estimates, b.estimates) and np.array_equal(a.ess, b.ess)


def test_eval_count_is_occupied_cells(cuda):
    frames, truth, init, dyn = _c1_like(n=10000, k=5)
    lik = _lik()
    r = pc.pcsir_track(frames, pc.PcFilterConfig(10000, init, dyn, RES, lik,
                                                 grid=pc.BinGrid.pixel_aligned(64, 64, 1)),
                       pc.PhiloxRng(1))
    assert r.likelihood_evals == lik.evals
    assert r.likelihood_evals < 10000 * len(frames) / 10


@pytest.mark.parametrize("n", [1, 2, 31, 257, 1023, 1025, 1793, 3841])
def test_fused_equals_general_at_ragged_sizes(cuda, n):
    # particle counts around warp / tile / resampling-tile boundaries
    # (32, 1024 step-1 tile, 1792 and 3840 resampler tiles) and N = 1
    frames, truth, init, dyn = _c1_like(k=4)
    g = pc.BinGrid.pixel_aligned(64, 64, 2)
    for fused_fn, cfg_fn in (
            (pc.pcsir_track, lambda lik: pc.PcFilterConfig(n, init, dyn, RES, lik, grid=g)),
            (pc.sir_track, lambda lik: pc.FilterConfig(n, init, dyn, RES, lik))):
        a = fused_fn(frames, cfg_fn(_lik()), pc.PhiloxRng(6), fused=True)
        b = fused_fn(frames, cfg_fn(_lik()), pc.PhiloxRng(6), fused=False)
        assert a.path == "fused" and b.path == "general"
        assert np.array_equal(a.estimates, b.estimates)
        assert np.array_equal(a.ess, b.ess)
        assert np.array_equal(a.resampled, b.resampled)


def test_pinned_host_frames_pipelined_upload(cuda):
    # a pinned float32 (K,H,W) host tensor is uploaded in chunks on a side
    # stream and filtered chunk by chunk: same result as device-resident frames
    from paper_1310_5541_b200 import synthesis as syn
    dev, truth = syn.spot_scene(9, 512, (203.0, 256.0), seed=2)
    host = dev.cpu().pin_memory()
    init = pc.InitSpec(pc.StateVector(203.0, 256.0, 0.5, 0.0, 20.0), "gauss", sigma=2.0)
    dyn = pc.DynamicsParams(0.5, 0.1, 1.0)
    g = pc.BinGrid.pixel_aligned(512, 512, 2)
    for res in (RES, pc.ResampleConfig(0.5, "systematic")):
        a = pc.pcsir_track(host, pc.PcFilterConfig(20000, init, dyn, res, _lik(), grid=g),
                           pc.PhiloxRng(3))
        b = pc.pcsir_track(dev, pc.PcFilterConfig(20000, init, dyn, res, _lik(), grid=g),
                           pc.PhiloxRng(3))
        assert a.path == b.path == "fused"
        assert np.array_equal(a.estimates, b.estimates)
        assert np.array_equal(a.resampled, b.resampled)


@pytest.mark.parametrize("frac", [1.0, 0.5])
@pytest.mark.parametrize("method", ["sir", "pc"])
def test_fused_multinomial_equals_general(cuda, frac, method):
    # multinomial resampling (filtering.py:96-97,100) in the fused loops: the
    # resampler writes the exact cdf, k_multinomial_emit searches the frame's
    # Philox points — bit-identical to the step-by-step driver
    frames, truth, init, dyn = _c1_like(n=3000, k=10)
    res = pc.ResampleConfig(frac, "multinomial")
    g = pc.BinGrid.pixel_aligned(64, 64, 2)

    def run(fused):
        lik = _lik()
        if method == "sir":
            return pc.sir_track(frames, pc.FilterConfig(3000, init, dyn, res, lik),
                                pc.PhiloxRng(12), fused=fused), lik
        return pc.pcsir_track(frames, pc.PcFilterConfig(3000, init, dyn, res, lik, grid=g),
                              pc.PhiloxRng(12), fused=fused), lik

    (a, la), (b, lb) = run(True), run(False)
    assert a.path == "fused" and b.path == "general"
    assert np.any(a.resampled)
    assert np.array_equal(a.resampled, b.resampled)
    assert np.array_equal(a.estimates, b.estimates)
    assert np.array_equal(a.ess, b.ess)
    assert la.evals == lb.evals


def test_capacity_fallback_with_prior_weights(cuda):
    """More occupied cells than the fused loop holds (MAXM = 2^20) on a frame
    whose particles carry prior weights (ESS threshold, no resampling): the
    fused loop stops cleanly (no second finalisation of the frame, no writes
    past the output rows) and the driver reruns the track on the general
    path (binning.py:212-226 semantics either way)."""
    n = 1_500_000
    frames, truth, init, _ = _c1_like(n=n, k=6)
    init = pc.InitSpec(pc.StateVector(32.0, 32.0, 0.0, 0.0, 20.0), "gauss", sigma=1.0)
    dyn = pc.DynamicsParams(2.0, 0.1, 1.0)
    res = pc.ResampleConfig(0.001, "systematic")
    grid = pc.BinGrid.pixel_aligned(64, 64, 200)          # 0.005 px cells, 1.6e8 cells
    flat = pc.SpotLikelihood(pc.PsfParams(1.5, 10.0), pc.LikelihoodParams(1e4, 5))
    flat2 = pc.SpotLikelihood(pc.PsfParams(1.5, 10.0), pc.LikelihoodParams(1e4, 5))
    a = pc.pcsir_track(frames, pc.PcFilterConfig(n, init, dyn, res, flat, grid=grid),
                       pc.PhiloxRng(13), fused=True)
    b = pc.pcsir_track(frames, pc.PcFilterConfig(n, init, dyn, res, flat2, grid=grid),
                       pc.PhiloxRng(13), fused=False)
    assert a.path == "general"            # the fused loop hit its capacity and fell back
    assert not a.resampled[1:].any()      # frames after the first carry prior weights
    assert np.array_equal(a.estimates, b.estimates)
    assert np.array_equal(a.ess, b.ess)
    assert a.likelihood_evals == b.likelihood_evals


@pytest.mark.parametrize("frac", [1.0, 0.3])
def test_fused_weighted_com_equals_general(cuda, frac):
    """pc_sis_step(weighted_com=True) (binning.py:160-165,186) in the fused
    loop: with uniform prior weights (every frame resampled) the weighted
    centre of mass is computed in the bins kernel from the exact cell sums;
    frames whose particles carry unequal prior weights (ESS threshold < 1)
    hand the track to the general path. Either way == the general driver."""
    frames, truth, init, dyn = _c1_like(n=3000, k=10)
    res = pc.ResampleConfig(frac, "systematic")
    grid = pc.BinGrid.pixel_aligned(64, 64, 2)
    cfg = pc.PcFilterConfig(3000, init, dyn, res, _lik(), grid=grid, weighted_com=True)
    a = pc.pcsir_track(frames, cfg, pc.PhiloxRng(8), fused=True)
    cfg2 = pc.PcFilterConfig(3000, init, dyn, res, _lik(), grid=grid, weighted_com=True)
    b = pc.pcsir_track(frames, cfg2, pc.PhiloxRng(8), fused=False)
    assert b.path == "general"
    if frac == 1.0:
        assert a.path == "fused"
    assert np.array_equal(a.estimates, b.estimates)
    assert np.array_equal(a.ess, b.ess)
    assert np.array_equal(a.resampled, b.resampled)
