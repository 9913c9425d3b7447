"""Pin the CPU oracle (oracle/) against golden vectors produced by the
reference itself (tests/golden/make_golden.py), Random123 known answers and
the reference tests' inline known answers. CPU only."""

import numpy as np
import pytest

from conftest import assert_propagation_close, golden
from oracle import pcsir_oracle as orc


# --- Philox4x32-10 known-answer vectors (Random123 kat_vectors) ---------------
@pytest.mark.parametrize("seed,ctr,want", [
    (0, [0, 0, 0, 0], [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]),
    (0xffffffffffffffff, [0xffffffff] * 4, [0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd]),
    (0x299f31d0a4093822, [0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344],
     [0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1]),
])
def test_philox_known_answers(seed, ctr, want):
    assert list(orc.philox4x32(seed, ctr)[0]) == want


def test_normals_law():
    # five normals per particle from one Philox block (three Box-Muller pairs,
    # the third one built from the leftover low bits): each column N(0, 1),
    # columns uncorrelated
    z = orc.propagate_normals(5, 0, 200_000)
    assert abs(z.mean()) < 0.005
    assert abs(z.std() - 1.0) < 0.005
    import scipy.stats
    for c in range(5):
        assert abs(z[c].std() - 1.0) < 0.01
        assert scipy.stats.kstest(z[c], "norm").pvalue > 1e-3
    cc = np.corrcoef(z)
    assert np.max(np.abs(cc - np.eye(5))) < 0.01
    assert np.max(np.abs(z)) < 5.7   # 22-bit u1: |z| <= sqrt(-2 ln 2^-23)


# --- likelihood operator (_speedups.pyx / kernels.py) --------------------------
@pytest.mark.parametrize("hw", [0, 4, 5, 7, 32])
def test_ssd_matches_reference(hw):
    g = golden("ssd")
    got = orc.spot_window_ssd(g["w_frame"], g["w_xs"], g["w_ys"], g["w_i0s"], 1.16, 10.0, hw)
    np.testing.assert_allclose(got, g[f"w_ssd_hw{hw}"], rtol=1e-12, atol=1e-12)


def test_ssd_brute_force_case():
    g = golden("ssd")
    got = orc.spot_window_ssd(g["b_frame"], g["b_xs"], g["b_ys"], g["b_i0s"], 1.5, 10.0, 3)
    np.testing.assert_allclose(got, g["b_ssd"], rtol=1e-12)
    py = orc.spot_window_ssd_py(g["b_frame"], g["b_xs"], g["b_ys"], g["b_i0s"], 1.5, 10.0, 3)
    np.testing.assert_allclose(py, g["b_ssd"], rtol=1e-12)


def test_reference_compiled_kernel_if_built():
    k = orc.reference_ssd_kernel()
    if k is None:
        pytest.skip("oracle/_ref not built")
    g = golden("ssd")
    got = k(g["w_frame"], g["w_xs"], g["w_ys"], g["w_i0s"], 1.16, 10.0, 4)
    assert np.array_equal(got, orc.spot_window_ssd(g["w_frame"], g["w_xs"], g["w_ys"],
                                                   g["w_i0s"], 1.16, 10.0, 4))


# --- partition / dummies (binning.py:97-112,157-172) ---------------------------
def _cases():
    return [str(c) for c in golden("partition")["cases"]]


@pytest.mark.parametrize("case", ["unit", "px1", "px4", "px2", "tiny"])
def test_partition_matches_reference(case):
    g = golden("partition")
    grid = tuple(g[f"{case}_grid"])
    grid = grid[:4] + (int(grid[4]), int(grid[5]))
    flat, order, unique, starts, counts = orc.partition(g[f"{case}_states"], grid)
    for name, got in (("flat", flat), ("order", order), ("unique", unique), ("starts", starts),
                      ("counts", counts)):
        assert np.array_equal(got, g[f"{case}_{name}"]), name


@pytest.mark.parametrize("case", ["unit", "px1", "px4", "px2", "tiny"])
def test_dummies_match_reference(case):
    g = golden("partition")
    grid = tuple(g[f"{case}_grid"])
    grid = grid[:4] + (int(grid[4]), int(grid[5]))
    st = g[f"{case}_states"]
    order, unique, starts, counts = (g[f"{case}_{k}"] for k in ("order", "unique", "starts", "counts"))
    for pl in ("com", "coc"):
        got = orc.dummy_states(st, grid, order, unique, starts, counts, pl)
        assert np.array_equal(got, g[f"{case}_dummies_{pl}"])
    got = orc.dummy_states(st, grid, order, unique, starts, counts, "com",
                           g[f"{case}_weights"][order])
    assert np.array_equal(got, g[f"{case}_dummies_wcom"])


@pytest.mark.parametrize("case", ["unit", "px1", "px4", "px2", "tiny"])
def test_canonical_dummies_vs_reference(case):
    """Exact-sum dummies equal the reference's reduceat means to float32
    rounding; singleton bins reproduce their member bit for bit."""
    g = golden("partition")
    st = g[f"{case}_states"]
    order, counts = g[f"{case}_order"], g[f"{case}_counts"]
    n = st.shape[0]
    bin_of = orc.bin_of_from_partition(n, order, counts)
    soa = st.T.astype(np.float32)
    d = orc.dummies_exact(soa, bin_of, counts).astype(np.float64).T
    ref = g[f"{case}_dummies_com"]
    np.testing.assert_allclose(d, ref, rtol=1e-6, atol=1e-6)
    single = counts == 1
    members = order[np.cumsum(counts) - 1][single]
    assert np.array_equal(d[single], st[members])
    # golden wcom = pc_sis_step's call: _dummy_states(..., weights[order]),
    # which the reference indexes by order again -> particle i weighs w[order[i]]
    w = g[f"{case}_weights"].astype(np.float32)
    dw = orc.dummies_exact(soa, bin_of, counts, prior_w=w[order]).astype(np.float64).T
    np.testing.assert_allclose(dw, g[f"{case}_dummies_wcom"], rtol=1e-6, atol=1e-6)


# --- filtering (normalize / ESS / resampling) ----------------------------------
@pytest.mark.parametrize("k", ["halves", "zeros", "tiny", "rand1000", "peaked"])
def test_normalize_and_ess_match_reference(k):
    g = golden("filtering")
    w = orc.normalize(g[f"norm_{k}_in"])
    assert np.array_equal(w, g[f"norm_{k}_out"])
    assert orc.effective_sample_size(w) == g[f"norm_{k}_ess"]
    # canonical (log-domain, exact normaliser) agrees to float32 rounding
    with np.errstate(divide="ignore"):
        w32, _, _ = orc.normalize_exact(np.log(g[f"norm_{k}_in"]))
    np.testing.assert_allclose(w32, g[f"norm_{k}_out"], rtol=2e-7, atol=1e-30)


@pytest.mark.parametrize("k", ["r10", "r1000", "r20000"])
def test_resample_indices_match_reference(k):
    g = golden("filtering")
    w, u = g[f"{k}_w"], float(g[f"{k}_u"])
    n = w.shape[0]
    ref = orc.resample_indices_reference(w.copy(), n, "systematic",
                                         orc.ReplayRng(randoms=[u]))
    assert np.array_equal(ref, g[f"{k}_sys"])
    # the canonical exact-prefix variant equals the reference at these sizes
    assert np.array_equal(orc.systematic_exact(w.astype(np.float32), u), g[f"{k}_sys"])
    assert np.array_equal(orc.multinomial_exact(w.astype(np.float32), g[f"{k}_pts"]),
                          g[f"{k}_mult"])


def test_zero_weight_never_selected():
    g = golden("filtering")
    anc = orc.systematic_exact(g["zero_w"].astype(np.float32), 0.25)
    assert np.array_equal(anc, g["zero_sys"])
    assert not np.any(anc == 1)


def test_estimate_ess_canonical_vs_reference():
    g = golden("filtering")
    st, w = g["pm_states"], g["pm_w"]
    est, ess = orc.estimate_ess_exact(st.T.astype(np.float32), w.astype(np.float32))
    np.testing.assert_allclose(est, g["pm_mean"], rtol=1e-6)
    np.testing.assert_allclose(ess, g["pm_ess"], rtol=1e-6)


# --- propagation ----------------------------------------------------------------
def test_propagate_matches_reference():
    g = golden("propagate")
    dyn = g["dyn"]
    noise = np.array([dyn[0], dyn[0], dyn[1], dyn[1], dyn[2]])
    out = orc.propagate_array(g["states"], noise, dyn[3], g["normals"])
    assert np.array_equal(out, g["out"])
    s32, z32 = g["states"].T.astype(np.float32), g["normals"].T.astype(np.float32)
    f64o = orc.propagate_f64_order(s32, z32, *dyn)
    assert np.array_equal(f64o, g["out"].T.astype(np.float32))
    # the device's canonical float32 form agrees to 2 float32 ulps of the
    # operand scale (double rounding of x + vx dt; parameters split hi + lo)
    f32 = orc.propagate_f32(s32, z32, *dyn)
    assert_propagation_close(f32, g["out"].T, s32, z32, dyn)



# --- whole filter driver ------------------------------------------------------
@pytest.mark.parametrize("name,cpp", [("sir", None), ("pc1", 1), ("pc4", 4)])
def test_track_restatement_matches_reference(name, cpp):
    g = golden("tracks")
    frames = [f.astype(np.float64) for f in g["frames"]]
    h, w = frames[0].shape
    grid = None if cpp is None else (-0.5, -0.5, 1.0 / cpp, 1.0 / cpp, w * cpp, h * cpp)
    lik = orc.SpotModel(1.5, 10.0, 10.0, 5)
    est, ess, res, evals = orc.track(frames, int(g["n"]), g["init"], 2.0,
                                     [0.5, 0.5, 0.1, 0.1, 1.0], 1.0, lik,
                                     orc.PhiloxReplay(int(g["seed"])), grid=grid)
    assert np.array_equal(est, g[f"{name}_est"])
    assert np.array_equal(ess, g[f"{name}_ess"])
    assert np.array_equal(res, g[f"{name}_res"])
    assert evals == int(g[f"{name}_evals"])


# --- reference inline known answers (test_binning.py, test_imaging.py) ---------
def test_cell_index_examples():
    unit = (0.0, 0.0, 1.0, 1.0, 10, 10)
    assert orc.cell_indices([1.5], [2.5], unit) == ([1], [2])
    assert orc.cell_indices([1.0], [0.5], unit) == ([1], [0])       # lower-inclusive
    ix, iy = orc.cell_indices([-3.0, 99.0], [4.2, 4.2], unit)         # clamped
    assert list(ix) == [0, 9] and list(iy) == [4, 4]
    px = (-0.5, -0.5, 1.0, 1.0, 512, 512)
    assert orc.cell_indices(10.0, 20.0, px) == (10, 20)
    assert orc.cell_indices(10.49, 20.49, px) == (10, 20)
    assert orc.cell_indices(10.5, 20.5, px) == (11, 21)
    px2 = (-0.5, -0.5, 0.5, 0.5, 1024, 1024)
    assert orc.cell_indices(-0.3, -0.3, px2) == (0, 0)
    assert orc.cell_indices(0.3, -0.3, px2) == (1, 0)


def test_ssd_zero_for_perfect_prediction():
    sigma, bg = 2.0, 5.0
    ys, xs = np.mgrid[0:32, 0:32]
    frame = 20.0 * np.exp(-((xs - 14.0) ** 2) / (2 * sigma ** 2)) \
        * np.exp(-((ys - 17.0) ** 2) / (2 * sigma ** 2)) + bg
    ssd = orc.spot_window_ssd(frame, [14.0], [17.0], [20.0], sigma, bg, 4)
    assert ssd[0] == pytest.approx(0.0, abs=1e-18)


def test_poisson_models_sane():
    """R19 oracle self-consistency: erf model == pixel-integral of the Gaussian."""
    import math
    frame = np.full((32, 32), 10.0)
    ll = orc.loglik_poisson(frame, [16.2], [15.7], [0.0], 1.5, 10.0, 7, 1)
    assert ll[0] == 0.0                                   # no spot -> ratio 0
    frame2 = frame.copy()
    frame2[16, 16] = 30.0
    a = orc.loglik_poisson(frame2, [16.0], [16.0], [20.0], 1.5, 10.0, 7, 1)[0]
    b = orc.loglik_poisson(frame2, [5.0], [5.0], [20.0], 1.5, 10.0, 7, 1)[0]
    assert a > b
    s2 = math.sqrt(2) * 1.5
    ex = 1.5 * math.sqrt(math.pi / 2) * (math.erf(0.5 / s2) - math.erf(-0.5 / s2))
    mu = 20.0 * ex * ex
    single = orc.loglik_poisson(np.full((1, 1), 10.0), [0.0], [0.0], [20.0], 1.5, 10.0, 0, 1)[0]
    assert single == pytest.approx(10.0 * math.log1p(mu / 10.0) - mu, rel=1e-12)


# --- scene synthesis (synthesis.py:124-130) ------------------------------------
def test_render_ideal_matches_reference_golden():
    g = golden("synth")
    h, w = g["frames"].shape[1:]
    for s, f in zip(g["states"], g["frames"]):
        got = orc.render_ideal(s[[0, 1, 4]][None, :], w, h, float(g["sigma"]), float(g["bg"]))
        np.testing.assert_allclose(got, f, rtol=0, atol=1e-12)
