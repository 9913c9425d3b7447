"""Generate golden vectors for the pcSIR / SIR hot path by running the
UNMODIFIED reference package (/root/reference/pkg/src/pcsir) in this
container. The fixtures pin the oracle (tests/test_oracle_golden.py) and the
device path (tests/test_gpu_*.py); /root/reference is not needed at test time.

Run:  python tests/golden/make_golden.py      (writes tests/golden/*.npz)

All state / weight inputs are float32-representable so the float32 device
path can be compared bit-for-bit where the contract is bit-exact.
"""

import os
import pathlib
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
REPO = HERE.parents[1]
REF_SRC = pathlib.Path("/root/reference/pkg/src")

os.environ.setdefault("PCSIR_KERNELS", "python")  # the reference's numpy kernel (no build)
sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(REPO))

import pcsir  # noqa: E402  (reference)
from pcsir import binning as rb  # noqa: E402
from pcsir import filtering as rf  # noqa: E402
from pcsir import kernels as rk  # noqa: E402
from pcsir import state as rs  # noqa: E402
from pcsir import synthesis as rsyn  # noqa: E402
from pcsir.imaging import (ImageFrame, LikelihoodParams, PsfParams,  # noqa: E402
                           SpotLikelihood)

from oracle import pcsir_oracle as orc  # noqa: E402

# Use the reference's own compiled kernel (its default backend) when
# oracle/build_ref.sh has built it from /root/reference/pkg/src/pcsir/_speedups.pyx.
_compiled = orc.reference_ssd_kernel()
if _compiled is not None:
    rk._IMPLS["compiled"] = _compiled
    rk.set_backend("compiled")


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def workload(rng, n=200, shape=(64, 64)):
    """test_kernels.py:9-14 (_workload)."""
    frame = rng.poisson(12.0, size=shape).astype(np.float64)
    xs = rng.uniform(-5, shape[1] + 5, size=n)
    ys = rng.uniform(-5, shape[0] + 5, size=n)
    i0s = rng.uniform(0.0, 30.0, size=n)
    return frame, xs, ys, i0s


def gen_ssd():
    out = {}
    rng = np.random.default_rng(20240)  # conftest.py:9-11
    frame, xs, ys, i0s = workload(rng)
    xs, ys, i0s = f32(xs), f32(ys), f32(i0s)
    out["w_frame"], out["w_xs"], out["w_ys"], out["w_i0s"] = frame, xs, ys, i0s
    for hw in (0, 4, 5, 7, 32):
        out[f"w_ssd_hw{hw}"] = rk.spot_window_ssd(frame, xs, ys, i0s, 1.16, 10.0, hw)
    # c1 likelihood shape: sigma 1.5, hw 5
    out["w_ssd_c1"] = rk.spot_window_ssd(frame, xs, ys, i0s, 1.5, 10.0, 5)
    # brute force case (test_kernels.py:68-89)
    frame2, xs2, ys2, i2 = workload(np.random.default_rng(7), n=25, shape=(20, 20))
    xs2, ys2, i2 = f32(xs2), f32(ys2), f32(i2)
    out["b_frame"], out["b_xs"], out["b_ys"], out["b_i0s"] = frame2, xs2, ys2, i2
    out["b_ssd"] = rk.spot_window_ssd(frame2, xs2, ys2, i2, 1.5, 10.0, 3)
    return out


def gen_partition():
    out = {}
    rng = np.random.default_rng(11)
    cases = []
    # unit grid with out-of-grid states (test_binning.py:67-74 style)
    pos = f32(rng.uniform(-5, 15, size=(300, 2)))
    cases.append(("unit", pos, rb.BinGrid(0.0, 0.0, 1.0, 1.0, 10, 10)))
    # pixel grids around a spot, 1 and 4 cells per pixel
    cloud = f32(np.array([31.3, 30.7]) + rng.normal(0, 2.0, size=(2000, 2)))
    cases.append(("px1", cloud, rb.BinGrid.pixel_aligned(64, 64, 1)))
    cases.append(("px4", cloud, rb.BinGrid.pixel_aligned(64, 64, 4)))
    cases.append(("px2", cloud, rb.BinGrid.pixel_aligned(64, 64, 2)))
    # sub-spacing cells: 64-bit flat ids (test_binning.py:198-199)
    tiny_pos = f32(rng.uniform(18, 22, size=(64, 2)))
    cases.append(("tiny", tiny_pos, rb.BinGrid(-0.5, -0.5, 1e-6, 1e-6, 40 * 10 ** 6, 40 * 10 ** 6)))
    for name, xy, grid in cases:
        n = xy.shape[0]
        states = np.zeros((n, 5))
        states[:, :2] = xy
        states[:, 2:] = f32(rng.normal(0, 1, size=(n, 3)) * [0.5, 0.5, 3.0] + [0.1, -0.2, 20.0])
        flat, order, unique, starts, counts = rb._partition(states, grid)
        weights = f32(rng.uniform(0.1, 2.0, size=n))
        out[f"{name}_states"] = states
        out[f"{name}_grid"] = np.array([grid.origin_x, grid.origin_y, grid.cell_width,
                                        grid.cell_height, grid.n_cols, grid.n_rows])
        out[f"{name}_flat"] = flat
        out[f"{name}_order"] = order
        out[f"{name}_unique"] = unique
        out[f"{name}_starts"] = starts
        out[f"{name}_counts"] = counts
        out[f"{name}_weights"] = weights
        for placement in (rb.DummyPlacement.CENTER_OF_MASS, rb.DummyPlacement.CELL_CENTER):
            out[f"{name}_dummies_{placement.value}"] = rb._dummy_states(
                states, grid, order, unique, starts, counts, placement)
        out[f"{name}_dummies_wcom"] = rb._dummy_states(
            states, grid, order, unique, starts, counts, rb.DummyPlacement.CENTER_OF_MASS,
            weights[order])
    out["cases"] = np.array([c[0] for c in cases])
    return out


class Replay:
    def __init__(self, normals=(), randoms=()):
        self.normals = list(normals)
        self.randoms = list(randoms)

    def normal(self, loc=0.0, scale=1.0, size=None):
        return loc + scale * np.asarray(self.normals.pop(0)).reshape(size)

    def random(self, size=None):
        r = self.randoms.pop(0)
        return float(r) if size is None else np.asarray(r).reshape(size)


def gen_filtering():
    out = {}
    rng = np.random.default_rng(5)
    vecs = {
        "halves": [2.0, 2.0],
        "zeros": [0.0, 5.0],
        "tiny": [1e-300, 1e-300],
        "rand1000": rng.uniform(0, 1, size=1000),
        "peaked": np.exp(-rng.uniform(0, 40, size=5000)),
    }
    for k, v in vecs.items():
        v = np.asarray(v, dtype=np.float64)
        ps = rs.ParticleSet(np.zeros((len(v), 5)), v)
        nw = rf.normalize(ps).weights
        out[f"norm_{k}_in"] = v
        out[f"norm_{k}_out"] = nw
        out[f"norm_{k}_ess"] = rf.effective_sample_size(rf.normalize(ps))
    # resampling indices with the reference's sequential cumsum (filtering.py:93-100)
    for k, n in (("r10", 10), ("r1000", 1000), ("r20000", 20000)):
        w = f32(rng.uniform(0, 1, size=n) ** 3)
        w = f32(w / w.sum())
        u = float(rng.random())
        out[f"{k}_w"] = w
        out[f"{k}_u"] = u
        out[f"{k}_sys"] = rf._resample_indices(w.copy(), n, "systematic", Replay(randoms=[u]))
        pts = rng.random(n)
        out[f"{k}_pts"] = pts
        out[f"{k}_mult"] = rf._resample_indices(w.copy(), n, "multinomial", Replay(randoms=[pts]))
    # zero weights never selected (test_filtering.py:174-178)
    w = np.array([0.5, 0.0, 0.5], dtype=np.float64)
    out["zero_w"] = w
    out["zero_sys"] = rf._resample_indices(w.copy(), 3, "systematic", Replay(randoms=[0.25]))
    # posterior mean on a weighted set
    st = f32(rng.normal(10, 3, size=(500, 5)))
    w = f32(rng.uniform(0, 1, size=500))
    w = w / w.sum()
    out["pm_states"] = st
    out["pm_w"] = w
    out["pm_mean"] = rf.posterior_mean(rs.ParticleSet(st, w))
    out["pm_ess"] = rf.effective_sample_size(rs.ParticleSet(st, w))
    return out


def gen_propagate():
    out = {}
    rng = np.random.default_rng(9)
    n = 4000
    st = f32(np.column_stack([rng.uniform(0, 256, n), rng.uniform(0, 256, n),
                              rng.normal(0, 1, n), rng.normal(0, 1, n), rng.uniform(0, 40, n)]))
    st[:10, 4] = 0.0
    z = f32(rng.normal(size=(n, 5)))
    dyn = rs.DynamicsParams(0.5, 0.1, 1.0, 1.0)
    out["states"] = st
    out["normals"] = z
    out["dyn"] = np.array([0.5, 0.1, 1.0, 1.0])
    out["out"] = rs.propagate_array(st, dyn, Replay(normals=[z]))
    return out


def scene(seed_truth, seed_noise, width=48, height=48, frames=12):
    psf = PsfParams(1.5, 10.0)
    cfg = rsyn.SceneConfig(psf=psf, snr=4.0, frames=frames, width=width, height=height,
                           speed_min=0.5, speed_max=1.0, margin=8,
                           dynamics=rs.DynamicsParams(0.1, 0.1, 0.0))
    truth = rsyn.generate_truth(cfg, np.random.default_rng(seed_truth))
    frames_ = rsyn.render_sequence(truth, cfg, np.random.default_rng(seed_noise))
    return cfg, truth, frames_


def gen_tracks():
    out = {}
    cfg_scene, truth, frames = scene(3, 4)
    out["frames"] = np.stack([f.pixels for f in frames]).astype(np.float32)
    out["truth"] = truth.states
    out["init"] = truth.init_state
    seed = 1234
    n = 300
    init = rs.InitSpec(rs.StateVector.from_array(truth.init_state), "gauss", sigma=2.0)
    dyn = rs.DynamicsParams(0.5, 0.1, 1.0)
    res = rf.ResampleConfig(1.0, "systematic")
    for name, grid in (("sir", None), ("pc1", rb.BinGrid.pixel_aligned(48, 48, 1)),
                       ("pc4", rb.BinGrid.pixel_aligned(48, 48, 4))):
        lik = SpotLikelihood(cfg_scene.psf, LikelihoodParams(10.0, 5))
        if grid is None:
            r = rf.sir_track(frames, rf.FilterConfig(n, init, dyn, res, lik), orc.PhiloxReplay(seed))
        else:
            r = rb.pcsir_track(frames, rb.PcFilterConfig(n, init, dyn, res, lik, grid=grid),
                               orc.PhiloxReplay(seed))
        out[f"{name}_est"] = r.estimates
        out[f"{name}_ess"] = r.ess
        out[f"{name}_res"] = r.resampled
        out[f"{name}_evals"] = r.likelihood_evals
    out["seed"] = seed
    out["n"] = n
    return out


def gen_steps():
    """pc_sis_step / sis_step on fixed float32 inputs with replayed normals."""
    out = {}
    rng = np.random.default_rng(21)
    cfg_scene, truth, frames = scene(5, 6, frames=1)
    frame = frames[0]
    n = 1500
    st = f32(np.column_stack([truth.states[0, 0] + rng.normal(0, 1.5, n),
                              truth.states[0, 1] + rng.normal(0, 1.5, n),
                              rng.normal(0.5, 0.2, n), rng.normal(0, 0.2, n),
                              rng.normal(truth.states[0, 4], 2.0, n)]))
    w = f32(rng.uniform(0.5, 1.5, n))
    z = f32(rng.normal(size=(n, 5)))
    dyn = rs.DynamicsParams(0.5, 0.1, 1.0)
    lik = SpotLikelihood(cfg_scene.psf, LikelihoodParams(10.0, 5))
    out["frame"] = frame.pixels
    out["states"] = st
    out["weights"] = w
    out["normals"] = z
    ps = rs.ParticleSet(st, w)
    s1 = rf.sis_step(ps, frame, lik, dyn, Replay(normals=[z]))
    out["sis_states"], out["sis_weights"] = s1.states, s1.weights
    for cpp in (1, 2, 4):
        grid = rb.BinGrid.pixel_aligned(frame.width, frame.height, cpp)
        lik = SpotLikelihood(cfg_scene.psf, LikelihoodParams(10.0, 5))
        s2, occ = rb.pc_sis_step(rs.ParticleSet(st, w), frame, lik, dyn, grid,
                                 rb.DummyPlacement.CENTER_OF_MASS, Replay(normals=[z]))
        out[f"pc{cpp}_states"], out[f"pc{cpp}_weights"] = s2.states, s2.weights
        out[f"pc{cpp}_occ"] = occ
        out[f"pc{cpp}_evals"] = lik.evals
    return out


def gen_synth():
    """render_clean_frame (synthesis.py:124-130) of the unmodified reference
    for states in the interior, at a border and off the frame."""
    from pcsir import synthesis as rsyn
    from pcsir.imaging import PsfParams as RPsf
    cfg = rsyn.SceneConfig(psf=RPsf(1.5, 10.0), snr=4.0, frames=1, width=48, height=40)
    states = np.array([[20.3, 17.6, 0.0, 0.0, 20.0], [0.4, 39.2, 0.0, 0.0, 35.5],
                       [47.9, 3.3, 0.0, 0.0, 12.25], [-3.0, 50.0, 0.0, 0.0, 8.0]])
    frames = np.stack([rsyn.render_clean_frame(s, cfg) for s in states])
    return {"states": states, "frames": frames, "sigma": 1.5, "bg": 10.0}


def gen_bounds():
    """bounds.py:121-180 and experiments.py:370-388 on the reference."""
    from pcsir import bounds as rbd
    from pcsir import experiments as rex
    out = {}
    fields = {"quadratic": rbd.quadratic_field(), "linear": rbd.linear_field(),
              "sinsin": rbd.sinsin_field(), "gaussian": rbd.gaussian_spot_field(),
              "gauss2": rbd.gaussian_spot_field(1.5, 20.0, 10.0, (0.3, -0.2))}
    domains = {"quadratic": (0.0, 4.0, 0.0, 4.0), "linear": (0.0, 1.0, 0.0, 1.0),
               "sinsin": (0.0, np.pi, 0.0, np.pi), "gaussian": (-4.0, 4.0, -4.0, 4.0),
               "gauss2": (-3.0, 5.0, -4.0, 2.0)}
    rng = np.random.default_rng(5)
    for name, fld in fields.items():
        dom = domains[name]
        for cells in ((4, 4), (7, 3), (16, 16), (33, 20)):
            part = rbd.DomainPartition.uniform(dom, *cells)
            key = f"{name}_{cells[0]}x{cells[1]}"
            out[f"{key}_dmax"] = np.array(rbd.derivative_maxima(fld, part))
            out[f"{key}_rect"] = np.array(rbd.rect_bound(fld, part))
            out[f"{key}_mid64"] = np.array(rbd.midpoint_error(fld, part))
            out[f"{key}_mid16"] = np.array(rbd.midpoint_error(fld, part, quad_points=16))
        xe = np.sort(np.concatenate(([dom[0], dom[1]], rng.uniform(dom[0], dom[1], 9))))
        ye = np.sort(np.concatenate(([dom[2], dom[3]], rng.uniform(dom[2], dom[3], 6))))
        part = rbd.DomainPartition(xe, ye)
        out[f"{name}_irr_x"], out[f"{name}_irr_y"] = xe, ye
        out[f"{name}_irr_dmax"] = np.array(rbd.derivative_maxima(fld, part))
        out[f"{name}_irr_rect"] = np.array(rbd.rect_bound(fld, part))
        out[f"{name}_irr_mid64"] = np.array(rbd.midpoint_error(fld, part))
    for name, rows in rex.run_bounds_study().items():
        out[f"study_{name}"] = np.array(rows)
    return out


def gen_experiments():
    """The reference's tracking sweep (experiments.py:251-292) on a reduced
    small_object preset, with the scenes it rendered (derive_rng 'scene'
    streams), so the device harness can run on the same frames."""
    from dataclasses import replace
    import types
    if "matplotlib" not in sys.modules:   # reports.py imports it for plotting only (absent here)
        mpl = types.ModuleType("matplotlib")
        mpl.use = lambda *a, **k: None
        plt = types.ModuleType("matplotlib.pyplot")
        plt.rcParams = {}
        mpl.pyplot = plt
        sys.modules["matplotlib"] = mpl
        sys.modules["matplotlib.pyplot"] = plt
    from pcsir import experiments as rex
    from pcsir import reports as rrep
    from pcsir import synthesis as rsy
    cfg = rex.preset("small_object", seed=3)
    cfg = replace(cfg, n_particles=(2000, 8000), repetitions=8,
                  scene=replace(cfg.scene, frames=20, width=64, height=64))
    records = rex.run_tracking_experiment(cfg)
    rows = rrep.summarize(records)
    out = {"variants": np.array(cfg.variants), "n_particles": np.array(cfg.n_particles),
           "sigma_psf": np.array(cfg.scene.psf.sigma_psf), "i_bg": np.array(cfg.scene.psf.i_bg),
           "sigma_xi": np.array(cfg.sigma_xi), "hw": np.array(cfg.window_halfwidth),
           "filter_dyn": np.array([cfg.filter_dynamics.sigma_pos, cfg.filter_dynamics.sigma_vel,
                                   cfg.filter_dynamics.sigma_int, cfg.filter_dynamics.dt]),
           "prior": np.array(cfg.prior),
           "summary_columns": np.array(rrep.SUMMARY_COLUMNS)}
    for rep in range(cfg.repetitions):
        rng = rex.derive_rng(cfg.seed, "scene", cfg.experiment, rep)
        truth = rsy.generate_truth(cfg.scene, rng)
        frames = rsy.render_sequence(truth, cfg.scene, rng)
        out[f"frames_{rep}"] = np.stack([f.pixels for f in frames]).astype(np.uint16)
        out[f"positions_{rep}"] = truth.positions
        out[f"init_{rep}"] = truth.init_state
    out["rec_variant"] = np.array([r.variant for r in records])
    out["rec_n"] = np.array([r.n_particles for r in records])
    out["rec_rmse"] = np.array([r.rmse for r in records])
    out["rec_evals"] = np.array([r.lik_evals for r in records])
    out["rec_failed"] = np.array([r.failed for r in records])
    out["sum_variant"] = np.array([r.variant for r in rows])
    out["sum_n"] = np.array([r.n_particles for r in rows])
    out["sum_rmse_mean"] = np.array([r.rmse_mean for r in rows])
    out["sum_evals_mean"] = np.array([r.lik_evals_mean for r in rows])
    return out


def main():
    if len(sys.argv) > 1:   # regenerate the named fixtures only
        for name in sys.argv[1:]:
            np.savez_compressed(HERE / f"{name}.npz", **globals()[f"gen_{name}"]())
        return
    np.savez_compressed(HERE / "ssd.npz", **gen_ssd())
    np.savez_compressed(HERE / "partition.npz", **gen_partition())
    np.savez_compressed(HERE / "filtering.npz", **gen_filtering())
    np.savez_compressed(HERE / "propagate.npz", **gen_propagate())
    np.savez_compressed(HERE / "steps.npz", **gen_steps())
    np.savez_compressed(HERE / "tracks.npz", **gen_tracks())
    np.savez_compressed(HERE / "synth.npz", **gen_synth())
    for p in sorted(HERE.glob("*.npz")):
        print(p.name, p.stat().st_size)
    print("reference backend:", rk.active_backend(), "pcsir", pcsir.__version__)


if __name__ == "__main__":
    main()
