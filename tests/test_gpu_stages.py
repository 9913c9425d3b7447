"""Stage-wise parity of the device filter step against the CPU oracle
(SURVEY §8c protocol): every stage runs on the device's own float32 inputs
and the device's own RNG draws; bin ids, counts, dummies, ancestors,
estimates and ESS are compared bit-for-bit, likelihoods / weights within the
north-star 1e-5 tolerance."""

import ctypes

import numpy as np
import pytest
import torch

import paper_1310_5541_b200 as pc
from conftest import assert_propagation_close, golden, spot_pixels
from oracle import pcsir_oracle as orc
from paper_1310_5541_b200 import _lib, binning, filtering, kernels, state

pytestmark = pytest.mark.gpu

LOGLIK_TOL = 1e-5   # |d log L| <= 1e-5  <=>  likelihood / weight relative error <= 1e-5
W_RTOL = 1e-5


def _grid_tuple(g):
    return (g.origin_x, g.origin_y, g.cell_width, g.cell_height, g.n_cols, g.n_rows)


# --- RNG ---------------------------------------------------------------------------
def test_device_normals_match_philox_restatement(cuda):
    seed = 987654321
    for frame, n, off in ((0, 10000, 0), (7, 3000, 2 ** 33 + 5)):
        dev = state.device_normals(seed, frame, n, offset=off).double().cpu().numpy()
        ref = orc.propagate_normals(seed, frame, n, offset=off)
        # same Philox words; float32 SFU Box-Muller (__logf/__sincosf, ~2^-21
        # absolute) vs the float64 restatement
        assert np.max(np.abs(dev - ref)) < 1e-4
        assert np.max(np.abs(dev - ref) / np.maximum(1.0, np.abs(ref))) < 2e-5
        assert np.median(np.abs(dev - ref)) < 5e-7


def test_device_normals_law(cuda):
    import scipy.stats
    z = state.device_normals(3, 0, 500_000).double().cpu().numpy()
    for c in range(5):
        assert abs(z[c].mean()) < 0.006
        assert abs(z[c].std() - 1.0) < 0.006
    assert scipy.stats.kstest(z[2], "norm").pvalue > 1e-4
    assert abs(np.corrcoef(z[0], z[1])[0, 1]) < 0.01


def test_resample_u_host_equals_oracle(cuda):
    r = pc.PhiloxRng(55)
    for f in (0, 1, 99):
        assert r.resample_u(f) == orc.resample_u(55, f)


# --- propagation (state.py:115-127) -------------------------------------------------
def test_propagate_bitexact_with_device_normals(cuda):
    rng = np.random.default_rng(1)
    n, seed = 100_000, 4242
    host = np.column_stack([rng.uniform(0, 256, n), rng.uniform(0, 256, n), rng.normal(0, 1, n),
                            rng.normal(0, 1, n), rng.uniform(0, 3, n)]).astype(np.float32)
    soa = torch.from_numpy(np.ascontiguousarray(host.T)).cuda()
    dyn = pc.DynamicsParams(0.5, 0.1, 1.0)
    out = state.propagate_array(soa, dyn, pc.PhiloxRng(seed))
    z = state.device_normals(seed, 0, n).cpu().numpy()
    want = orc.propagate_f32(host.T, z, 0.5, 0.1, 1.0, 1.0)
    assert np.array_equal(out.cpu().numpy(), want)
    assert out[4].min().item() >= 0.0
    # and within two float32 ulps of the reference's float64 order
    ref = orc.propagate_f64_order(host.T, z, 0.5, 0.1, 1.0, 1.0).astype(np.float64)
    assert_propagation_close(out.cpu().numpy(), ref, host.T, z, (0.5, 0.1, 1.0, 1.0))


def test_propagate_golden_replayed_normals(cuda):
    g = golden("propagate")
    d = g["dyn"]
    out = state.propagate_with_normals(g["states"], pc.DynamicsParams(d[0], d[1], d[2], d[3]),
                                       g["normals"].T)
    s32, z32 = g["states"].T.astype(np.float32), g["normals"].T.astype(np.float32)
    # bit-exact against the canonical float32 form, and close to the
    # reference's float64 values (reference golden, state.py:115-127)
    assert np.array_equal(out.cpu().numpy(), orc.propagate_f32(s32, z32, *d))
    assert_propagation_close(out.cpu().numpy(), g["out"].T, s32, z32, d)


def test_init_cloud_matches_oracle(cuda):
    seed, n = 31, 50_000
    init = pc.InitSpec(pc.StateVector(20.0, 32.0, 0.5, 0.0, 20.0), "gauss", sigma=2.0)
    ps = pc.init_particle_set(n, init, pc.PhiloxRng(seed))
    z = torch.empty((2, n), dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib().pcs_philox_init_normals(seed, 0, n, _lib.ptr(z), n, _lib.stream()))
    zz = z.double().cpu().numpy()
    want_x = (20.0 + 2.0 * zz[0]).astype(np.float32)
    want_y = (32.0 + 2.0 * zz[1]).astype(np.float32)
    got = ps.soa.cpu().numpy()
    assert np.array_equal(got[0], want_x) and np.array_equal(got[1], want_y)
    assert np.all(got[2] == 0.5) and np.all(got[4] == 20.0)
    assert ps.weights[0] == 1.0 / n
    assert abs(got[0].std() - 2.0) < 0.03


# --- likelihood operator ---------------------------------------------------------------
@pytest.mark.parametrize("hw", [0, 4, 5, 7, 32])
def test_ssd_operator_matches_reference_golden(cuda, hw):
    g = golden("ssd")
    got = kernels.spot_window_ssd(g["w_frame"], g["w_xs"], g["w_ys"], g["w_i0s"], 1.16, 10.0, hw)
    np.testing.assert_allclose(got, g[f"w_ssd_hw{hw}"], rtol=1e-12, atol=1e-12)


def test_ssd_operator_brute_force_golden(cuda):
    g = golden("ssd")
    got = kernels.spot_window_ssd(g["b_frame"], g["b_xs"], g["b_ys"], g["b_i0s"], 1.5, 10.0, 3)
    np.testing.assert_allclose(got, g["b_ssd"], rtol=1e-10)


@pytest.mark.parametrize("hw,sigma", [(4, 1.16), (5, 1.5), (7, 2.0), (32, 13.0), (9, 3.0)])
def test_loglik_f32_within_tolerance(cuda, hw, sigma):
    g = golden("ssd")
    frame = pc.ImageFrame(g["w_frame"])
    lik = pc.SpotLikelihood(pc.PsfParams(sigma, 10.0), pc.LikelihoodParams(10.0, hw))
    soa = torch.from_numpy(np.ascontiguousarray(np.stack(
        [g["w_xs"], g["w_ys"], np.zeros(200), np.zeros(200), g["w_i0s"]]).astype(np.float32))).cuda()
    ll = lik.loglik(soa, frame).double().cpu().numpy()
    ref = orc.loglik_gauss(g["w_frame"], g["w_xs"], g["w_ys"], g["w_i0s"], sigma, 10.0, hw, 10.0)
    assert np.max(np.abs(ll - ref)) <= LOGLIK_TOL * max(1.0, (2 * hw + 1) ** 2 / 121)
    assert lik.evals == 200


def test_likelihood_exact_ones(cuda):
    psf = pc.PsfParams(1.16, 10.0)
    st = pc.StateVector(30.25, 31.75, 0.0, 0.0, 22.0)
    frame = pc.ImageFrame(spot_pixels(30.25, 31.75, 22.0, 1.16, 10.0))
    lik = pc.SpotLikelihood(psf, pc.LikelihoodParams(10.0, 4))
    assert lik(st, frame) == 1.0                            # test_imaging.py:32-36
    flat = pc.ImageFrame(np.full((32, 32), 10.0))
    assert lik(pc.StateVector(16.0, 16.0, 0, 0, 0.0), flat) == 1.0   # test_imaging.py:39-42
    soa = torch.tensor([[16.0], [16.0], [0.0], [0.0], [0.0]], device="cuda")
    assert lik.loglik(soa, flat).item() == 0.0
    far = lik(pc.StateVector(-100.0, -100.0, 0, 0, 0.0), flat)
    assert np.isfinite(far) and far > 0


def _poisson_term_mass(pix, xs, ys, i0s, sigma, bg, hw, model):
    """Per evaluation, sum over the window pixels (a superset: +-(hw + 1)
    around the rounded position, inside the frame) of |z log1p(mu/bg)| + |mu|
    in float64 — the scale of the float32 SIR form's rounding error bound
    (DESIGN.md §2)."""
    from scipy.special import erf
    h, w = pix.shape
    offs = np.arange(-hw - 1, hw + 2)
    out = np.empty(len(xs))
    for k, (x, y, i0) in enumerate(zip(xs.astype(np.float64), ys.astype(np.float64),
                                       i0s.astype(np.float64))):
        px = np.round(x).astype(int) + offs
        py = np.round(y).astype(int) + offs
        px, py = px[(px >= 0) & (px < w)], py[(py >= 0) & (py < h)]

        def axis(idx, p):
            if model == 1:
                c = np.sqrt(2.0) * sigma
                return sigma * np.sqrt(np.pi / 2) * (erf((idx + 0.5 - p) / c) - erf((idx - 0.5 - p) / c))
            sub = idx[:, None] - 0.375 + 0.25 * np.arange(4)[None, :] - p
            return np.mean(np.exp(-sub ** 2 / (2 * sigma ** 2)), axis=1)

        mu = i0 * np.outer(axis(py, y), axis(px, x))
        z = pix[np.ix_(py, px)]
        with np.errstate(invalid="ignore", divide="ignore"):
            lz = np.where(mu / bg > -1.0, np.abs(z * np.log1p(mu / bg)), np.inf)
        out[k] = np.sum(lz + np.abs(mu))
    return out


# float32 SIR Poisson form: |d log L| <= C 2^-24 sum_window (|z log1p(t)| + |mu|)
# (t = mu/bg to <= 28 ulp, log1p_pos 2 ulp, fma / product 2 ulp,
# a float32 row of <= 15 terms 14 ulp of its magnitude: 46 -> C = 64)
SIR_POISSON_C = 64.0


def test_poisson_loglik_matches_oracle(cuda):
    """R19 (config 3, builder-defined): the pcSIR per-cell form (float64,
    what the fused and general pcSIR paths evaluate for every dummy) meets
    |d log L| <= 1e-5 absolute against the float64 sub-pixel oracle; the
    per-particle SIR comparison form keeps float32 pixel terms (log L up to
    ~200 nats; 225 float32 terms of up to ~60 each) and meets the derived
    per-window bound C 2^-24 sum |term scale|, which is also
    within 4e-5 max(1, |log L|)."""
    rng = np.random.default_rng(3)
    pix = rng.poisson(spot_pixels(40.3, 38.8, 20.0, 1.5, 10.0, 96, 96)).astype(np.float64)
    n = 2000
    xs = rng.uniform(-3, 99, n).astype(np.float32)
    ys = rng.uniform(-3, 99, n).astype(np.float32)
    xs[:1000] = (40.3 + rng.normal(0, 1.5, 1000)).astype(np.float32)
    ys[:1000] = (38.8 + rng.normal(0, 1.5, 1000)).astype(np.float32)
    i0 = rng.uniform(5, 40, n).astype(np.float32)
    i0[1000:1020] = -2.0   # negative intensities take the library-log1p form
    soa = torch.from_numpy(np.stack([xs, ys, np.zeros(n, np.float32), np.zeros(n, np.float32),
                                     i0])).cuda()
    for sub, model in (("erf", 1), ("midpoint4", 2)):
        lik = pc.PoissonSpotLikelihood(pc.PsfParams(1.5, 10.0), pc.LikelihoodParams(10.0, 7), sub)
        ref = orc.loglik_poisson(pix, xs, ys, i0, 1.5, 10.0, 7, model)
        cells = lik.loglik(soa, pc.ImageFrame(pix), cells=True).double().cpu().numpy()
        assert np.max(np.abs(cells - ref)) <= LOGLIK_TOL, np.max(np.abs(cells - ref))
        fast = lik.loglik(soa, pc.ImageFrame(pix)).double().cpu().numpy()
        err = np.abs(fast - ref)
        bound = SIR_POISSON_C * 2.0 ** -24 * _poisson_term_mass(pix, xs, ys, i0, 1.5, 10.0, 7, model)
        print(f"R19 SIR {sub}: max |d log L| {err.max():.3g}, max err / bound {np.max(err / bound):.3g}")
        assert np.all(err <= bound + 1e-12), np.max(err / (bound + 1e-300))
        assert np.max(err / np.maximum(1.0, np.abs(ref))) < 4e-5, np.max(err)


# --- binning + dummies (binning.py:97-112,157-172) ---------------------------------------
@pytest.mark.parametrize("case", ["unit", "px1", "px4", "px2", "tiny"])
def test_partition_bitexact_golden(cuda, case):
    g = golden("partition")
    gg = g[f"{case}_grid"]
    grid = pc.BinGrid(gg[0], gg[1], gg[2], gg[3], int(gg[4]), int(gg[5]))
    flat, order, unique, starts, counts = binning._partition(g[f"{case}_states"], grid)
    for name, got in (("flat", flat), ("order", order), ("unique", unique), ("starts", starts),
                      ("counts", counts)):
        assert np.array_equal(got, g[f"{case}_{name}"]), name


@pytest.mark.parametrize("case", ["unit", "px1", "px4", "px2", "tiny"])
def test_dummies_bitexact_canonical(cuda, case):
    g = golden("partition")
    gg = g[f"{case}_grid"]
    grid = pc.BinGrid(gg[0], gg[1], gg[2], gg[3], int(gg[4]), int(gg[5]))
    st = g[f"{case}_states"]
    soa = torch.from_numpy(np.ascontiguousarray(st.T.astype(np.float32))).cuda()
    part = binning.partition_device(soa, grid)
    order, counts = g[f"{case}_order"], g[f"{case}_counts"]
    bin_of = orc.bin_of_from_partition(st.shape[0], order, counts)
    assert np.array_equal(part.bin_of.cpu().numpy(), bin_of)
    for placement, gold in ((pc.DummyPlacement.CENTER_OF_MASS, "com"),
                            (pc.DummyPlacement.CELL_CENTER, "coc")):
        d = binning.dummy_states_device(soa, grid, part, placement).cpu().numpy()
        want = orc.dummies_exact(soa.cpu().numpy(), bin_of, counts)
        if gold == "coc":
            want[0] = g[f"{case}_dummies_coc"][:, 0].astype(np.float32)
            want[1] = g[f"{case}_dummies_coc"][:, 1].astype(np.float32)
        assert np.array_equal(d, want), placement
        np.testing.assert_allclose(d.T, g[f"{case}_dummies_{gold}"], rtol=1e-6, atol=1e-6)
    single = counts == 1
    d = binning.dummy_states_device(soa, grid, part, pc.DummyPlacement.CENTER_OF_MASS).cpu().numpy()
    members = order[np.cumsum(counts) - 1][single]
    assert np.array_equal(d.T[single], st[members].astype(np.float32))
    # weighted CoM as pc_sis_step calls it (double permutation, binning.py:160,183)
    w = g[f"{case}_weights"].astype(np.float32)
    pw = torch.from_numpy(w[order]).cuda()
    dw = binning.dummy_states_device(soa, grid, part, pc.DummyPlacement.CENTER_OF_MASS, pw)
    want_w = orc.dummies_exact(soa.cpu().numpy(), bin_of, counts, prior_w=w[order])
    assert np.array_equal(dw.cpu().numpy(), want_w)
    np.testing.assert_allclose(dw.cpu().numpy().T, g[f"{case}_dummies_wcom"], rtol=1e-6, atol=1e-6)


def test_partition_large_against_oracle(cuda):
    rng = np.random.default_rng(8)
    n = 1_000_000
    host = np.stack([100 + rng.normal(0, 6, n), 120 + rng.normal(0, 6, n), rng.normal(0, 1, n),
                     rng.normal(0, 1, n), 20 + rng.normal(0, 2, n)]).astype(np.float32)
    soa = torch.from_numpy(host).cuda()
    for cpp in (4, 1, 2):
        grid = pc.BinGrid.pixel_aligned(256, 256, cpp)
        part = binning.partition_device(soa, grid)
        flat, order, unique, starts, counts = orc.partition(host.T.astype(np.float64),
                                                            _grid_tuple(grid))
        assert np.array_equal(part.unique.cpu().numpy(), unique)
        assert np.array_equal(part.counts.cpu().numpy(), counts)
        assert np.array_equal(part.order.cpu().numpy(), order)
        d = binning.dummy_states_device(soa, grid, part, pc.DummyPlacement.CENTER_OF_MASS)
        bin_of = orc.bin_of_from_partition(n, order, counts)
        assert np.array_equal(d.cpu().numpy(), orc.dummies_exact(host, bin_of, counts))


@pytest.mark.parametrize("cell,n", [(1e-5, 3_000_000), (0.25, 2_500_000), (64.0, 1_000_000)])
def test_partition_radix_sort_against_numpy(cuda, cell, n):
    """The hand-written stable LSD radix sort (pcs_sort.cuh) behind the per-step
    partition: 46-bit keys (1e-5 px cells, 6 passes), 26-bit keys, and a
    few heavily shared keys (64 px cells: long runs, stability across tiles);
    order, unique, starts, counts and the per-particle flat ids equal numpy's
    stable argsort / unique (binning.py:97-112)."""
    rng = np.random.default_rng(int(n))
    host = np.stack([rng.uniform(0, 255, n), rng.uniform(0, 255, n), rng.normal(0, 1, n),
                     rng.normal(0, 1, n), rng.uniform(0, 40, n)]).astype(np.float32)
    host[:2, : n // 4] = host[:2, :1]          # a quarter of the particles share one cell
    soa = torch.from_numpy(host).cuda()
    cells = int(round(256 / cell))
    grid = pc.BinGrid(-0.5, -0.5, cell, cell, cells, cells)
    part = binning.partition_device(soa, grid)
    flat, order, unique, starts, counts = orc.partition(host.T.astype(np.float64), _grid_tuple(grid))
    assert np.array_equal(part.flat.cpu().numpy().view(np.uint64).astype(np.int64), flat)
    assert np.array_equal(part.order.cpu().numpy(), order)
    assert np.array_equal(part.unique.cpu().numpy().view(np.uint64).astype(np.int64), unique)
    assert np.array_equal(part.starts.cpu().numpy(), starts)
    assert np.array_equal(part.counts.cpu().numpy(), counts)
    bin_of = orc.bin_of_from_partition(n, order, counts)
    assert np.array_equal(part.bin_of.cpu().numpy(), bin_of)


# --- weights, estimate, ESS, resampling (filtering.py:75-114) -----------------------------
@pytest.mark.parametrize("k", ["halves", "zeros", "tiny", "rand1000", "peaked"])
def test_normalize_golden(cuda, k):
    g = golden("filtering")
    v = g[f"norm_{k}_in"]
    ps = pc.normalize(pc.ParticleSet(np.zeros((len(v), 5)), v))
    np.testing.assert_allclose(ps.weights, g[f"norm_{k}_out"], rtol=W_RTOL, atol=1e-30)
    with np.errstate(divide="ignore"):
        w32, _, _ = orc.normalize_exact(np.log(v))
    np.testing.assert_allclose(ps.w.cpu().numpy(), w32, rtol=2e-7, atol=1e-37)
    assert pc.effective_sample_size(ps) == pytest.approx(float(g[f"norm_{k}_ess"]), rel=W_RTOL)


def test_normalize_exact_halves(cuda):
    assert np.array_equal(pc.normalize(pc.ParticleSet(np.zeros((2, 5)), [2.0, 2.0])).weights,
                          [0.5, 0.5])
    assert np.array_equal(pc.normalize(pc.ParticleSet(np.zeros((2, 5)), [0.0, 5.0])).weights,
                          [0.0, 1.0])
    assert np.array_equal(pc.normalize(pc.ParticleSet(np.zeros((2, 5)), [1e-300, 1e-300])).weights,
                          [0.5, 0.5])
    with pytest.raises(pc.DegenerateWeightsError):
        pc.normalize(pc.ParticleSet(np.zeros((2, 5)), [0.0, 0.0]))


def test_estimate_ess_bitexact(cuda):
    g = golden("filtering")
    st, w = g["pm_states"], g["pm_w"].astype(np.float32)
    ps = pc.ParticleSet.from_device(torch.from_numpy(st.T.astype(np.float32)).cuda(),
                                    w=torch.from_numpy(w).cuda())
    est, ess = filtering._estimate_ess(ps)
    est_ref, ess_ref = orc.estimate_ess_exact(st.T.astype(np.float32), w)
    assert np.array_equal(est, est_ref) and ess == ess_ref
    np.testing.assert_allclose(est, g["pm_mean"], rtol=W_RTOL)
    assert ess == pytest.approx(float(g["pm_ess"]), rel=W_RTOL)
    assert pc.effective_sample_size(pc.ParticleSet(np.zeros((8, 5)))) == pytest.approx(8.0, rel=1e-6)


def _device_anc(w32, u):
    n = w32.shape[0]
    w = torch.from_numpy(w32).cuda()
    anc = torch.empty(n, dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib().pcs_resample_systematic(_lib.ctx(), _lib.ptr(w), n, u, _lib.ptr(anc),
                                                  _lib.stream()))
    return anc.cpu().numpy()


@pytest.mark.parametrize("k", ["r10", "r1000", "r20000"])
def test_systematic_golden(cuda, k):
    g = golden("filtering")
    w, u = g[f"{k}_w"].astype(np.float32), float(g[f"{k}_u"])
    assert np.array_equal(_device_anc(w, u), g[f"{k}_sys"])
    n = w.shape[0]
    wt = torch.from_numpy(w).cuda()
    pts = torch.from_numpy(g[f"{k}_pts"]).cuda()
    anc = torch.empty(n, dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib().pcs_resample_multinomial(_lib.ctx(), _lib.ptr(wt), n, _lib.ptr(pts),
                                                   _lib.ptr(anc), _lib.stream()))
    assert np.array_equal(anc.cpu().numpy(), g[f"{k}_mult"])


@pytest.mark.parametrize("n", [1, 2, 3, 4095, 4096, 4097, 100_003, 1_000_000, 4_000_000])
def test_systematic_bitexact_canonical(cuda, n):
    rng = np.random.default_rng(n)
    w = rng.uniform(0, 1, n) ** 4
    w[rng.uniform(size=n) < 0.2] = 0.0
    if w.sum() == 0:
        w[0] = 1.0
    w = (w / w.sum()).astype(np.float32)
    u = float(rng.random())
    got = _device_anc(w, u)
    want = orc.systematic_exact(w, u)
    assert np.array_equal(got, want)
    assert np.all(np.diff(got) >= 0)
    assert not np.any(w[got] == 0)
    # how many slots the reference's own sequential float64 cumsum would move
    ref = orc.resample_indices_reference(w.astype(np.float64), n, "systematic",
                                         orc.ReplayRng(randoms=[u]))
    assert np.mean(ref != got) < 1e-4


def test_cdf_exact_matches_oracle(cuda):
    rng = np.random.default_rng(2)
    n = 300_001
    w = (rng.uniform(0, 1, n) ** 2).astype(np.float32)
    w /= w.sum()
    wt = torch.from_numpy(w).cuda()
    cdf = torch.empty(n, dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib().pcs_cdf(_lib.ctx(), _lib.ptr(wt), n, _lib.ptr(cdf), _lib.stream()))
    assert np.array_equal(cdf.cpu().numpy(), orc.cdf_exact(w))


def test_resample_law(cuda):
    # marginal frequencies within 1% of the weights (test_filtering.py:144-156)
    w = np.array([0.7, 0.2, 0.1])
    ps = pc.ParticleSet(np.column_stack([np.arange(3.0), np.zeros((3, 3)), np.ones(3)]), w)
    for scheme in ("systematic", "multinomial"):
        rng = pc.PhiloxRng(11)
        counts = np.zeros(3)
        trials = 3000
        for _ in range(trials):
            anc = filtering.resample_indices(ps, pc.ResampleConfig(scheme=scheme), rng)
            counts += np.bincount(anc.cpu().numpy(), minlength=3)
        freq = counts / (3 * trials)
        assert np.all(np.abs(freq - w) < 0.01), (scheme, freq)


def test_resample_resets_weights(cuda):
    ps = pc.normalize(pc.ParticleSet(np.column_stack([np.arange(10.0), np.zeros((10, 4))]),
                                     np.arange(1.0, 11.0)))
    out = pc.resample(ps, pc.ResampleConfig(scheme="systematic"), pc.PhiloxRng(1))
    assert len(out) == 10
    assert np.all(out.weights == 0.1)
    deg = pc.ParticleSet(np.column_stack([np.arange(3.0), np.zeros((3, 4))]), [1.0, 0.0, 0.0])
    out = pc.resample(deg, pc.ResampleConfig(), pc.PhiloxRng(2))
    assert np.all(out.states[:, 0] == 0.0)


# --- make_dummy (binning.py:129-154), device float64 in the reference's orders ------
def test_make_dummy_known_answers(cuda):
    # test_binning.py:97-126
    members = [pc.StateVector(0.2, 0.2, 1.0, -1.0, 10.0), pc.StateVector(0.8, 0.8, 1.0, -1.0, 10.0)]
    d = pc.make_dummy(members, (0, 1, 0, 1), pc.DummyPlacement.CENTER_OF_MASS)
    assert d == pc.StateVector(0.5, 0.5, 1.0, -1.0, 10.0)
    m = pc.StateVector(3.7, -1.2, 0.5, 0.25, 7.5)
    assert pc.make_dummy([m], (3, 4, -2, -1), pc.DummyPlacement.CENTER_OF_MASS) == m
    d = pc.make_dummy([pc.StateVector(1.9, 3.1, 2.0, 0.0, 5.0)], (1.0, 2.0, 3.0, 4.0),
                      pc.DummyPlacement.CELL_CENTER)
    assert d == pc.StateVector(1.5, 3.5, 2.0, 0.0, 5.0)
    d = pc.make_dummy([pc.StateVector(0, 0, 0, 0, 0), pc.StateVector(1, 0, 0, 0, 0)], (0, 1, 0, 1),
                      pc.DummyPlacement.CENTER_OF_MASS, weights=[1.0, 3.0])
    assert d.x == 0.75
    with pytest.raises(ValueError):
        pc.make_dummy([], (0, 1, 0, 1), pc.DummyPlacement.CENTER_OF_MASS)


@pytest.mark.parametrize("n", [1, 7, 100, 1000, 5000])
def test_make_dummy_matches_reference_orders(cuda, n):
    rng = np.random.default_rng(n)
    rows = rng.normal(size=(n, 5)) * np.array([50, 50, 1, 1, 10]) + np.array([100, 80, 0, 0, 20])
    rows[:, 4] = np.abs(rows[:, 4])
    members = [pc.StateVector(*r) for r in rows]
    d = pc.make_dummy(members, (0, 1, 0, 1), pc.DummyPlacement.CENTER_OF_MASS)
    # np.add.reduceat over axis 0 / n (binning.py:144-147), bit for bit (numpy adds the
    # first row to the pairwise sum of the others, per column)
    want = np.add.reduceat(rows, [0], axis=0)[0] / n
    assert np.array_equal(d.as_array(), want)
    w = rng.uniform(0.1, 2.0, n)
    dw = pc.make_dummy(members, (0, 1, 0, 1), pc.DummyPlacement.CENTER_OF_MASS, weights=w)
    np.testing.assert_allclose(dw.as_array(), (w @ rows) / w.sum(), rtol=1e-13)
    # the weight total is numpy's pairwise sum bit for bit: unit rows expose it
    ones = [pc.StateVector(1.0, 1.0, 1.0, 1.0, 1.0)] * n
    du = pc.make_dummy(ones, (0, 1, 0, 1), pc.DummyPlacement.CENTER_OF_MASS, weights=w)
    seq = 0.0
    for v in w:
        seq += v
    assert du.x == seq / w.sum()
