"""GPU tracking sweeps and the likelihood micro-benchmark.

Device counterpart of the reference's experiment harness around the filter
step: ``run_tracking_experiment`` (experiments.py:251-292) runs every
(variant, N, repetition) of a sweep on one GPU-rendered sequence per
repetition and records the same per-run fields (``RunRecord``);
``summarize`` / ``write_summary_csv`` collapse them into the reference's
summary columns (reports.py:19-21, 53-91: ``lik_evals_mean``,
``speedup_vs_sir`` ...); ``likelihood_benchmark`` is the ``backends``
micro-benchmark of cli.py:191-213 for the device likelihood operator.

Differences: frames come from ``synthesis.render_sequence`` (device Poisson
stream, not numpy's), the filters draw from ``PhiloxRng`` keyed by the same
order-independent (seed, tags) hash as the reference's ``derive_rng``, and
wall time covers the filtering call including the frame upload.
"""

import hashlib
import math
import time
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from .binning import (BinGrid, DummyPlacement, PcFilterConfig, dummy_states_device,
                      partition_device, pcsir_track)
from .filtering import (DegenerateWeightsError, FilterConfig, ResampleConfig, _check_not_degenerate,
                        _evaluate_loglik, _weight_update, normalize, posterior_mean, sir_track)
from .imaging import ImageFrame, LikelihoodParams, PsfParams, SpotLikelihood
from .kernels import spot_window_ssd
from .rng import PhiloxRng
from .state import DynamicsParams, InitSpec, ParticleSet, StateVector, init_particle_set
from . import synthesis as syn

VARIANT_LABELS = ("SIR", "pcSIR-1x1-CoM", "pcSIR-1x1-CoC", "pcSIR-2x2-CoM", "pcSIR-2x2-CoC")
SUMMARY_COLUMNS = ("experiment", "variant", "n_particles", "rmse_mean", "rmse_std",
                   "time_mean_s", "time_std_s", "lik_evals_mean", "speedup_vs_sir")


class ConfigError(ValueError):
    """Invalid experiment configuration (the reference's CLI exit code 2)."""


@dataclass(frozen=True)
class VariantSpec:
    """A parsed filter variant: SIR or a binned variant (experiments.py:41-50)."""

    label: str
    cells_per_pixel: int = None
    placement: DummyPlacement = None

    @property
    def is_pc(self):
        return self.cells_per_pixel is not None


def parse_variant(label) -> VariantSpec:
    """'SIR' or 'pcSIR-<c>x<c>[-com|-coc]' (experiments.py:53-71)."""
    token = label.strip().lower()
    if token == "sir":
        return VariantSpec("SIR")
    parts = token.split("-")
    if parts[0] != "pcsir" or len(parts) not in (2, 3):
        raise ConfigError(f"unknown filter variant {label!r}")
    a, _, b = parts[1].partition("x")
    if not (a.isdigit() and a == b and int(a) >= 1):
        raise ConfigError(f"unknown cell subdivision in variant {label!r}")
    try:
        placement = DummyPlacement(parts[2] if len(parts) == 3 else "com")
    except ValueError:
        raise ConfigError(f"unknown dummy placement in variant {label!r}") from None
    suffix = "CoM" if placement is DummyPlacement.CENTER_OF_MASS else "CoC"
    return VariantSpec(f"pcSIR-{a}x{a}-{suffix}", int(a), placement)


def derive_seed(seed, *tags):
    """Order-independent 64-bit key per tagged task (the hashing of
    experiments.py:93-99, folded to one Philox key)."""
    h = hashlib.sha256(repr((seed & 0xFFFFFFFF,) + tags).encode()).digest()
    return int.from_bytes(h[:8], "little")


@dataclass
class RunRecord:
    """One (variant, N, repetition) outcome (experiments.py:215-231)."""

    experiment: str
    variant: str
    n_particles: int
    repetition: int
    rmse: float
    wall_time_s: float
    lik_evals: int
    failed: bool = False
    trajectory: np.ndarray = None


@dataclass
class SummaryRow:
    experiment: str
    variant: str
    n_particles: int
    rmse_mean: float
    rmse_std: float
    time_mean_s: float
    time_std_s: float
    lik_evals_mean: float
    speedup_vs_sir: float


def generate_truth(width, height, frames, margin, i0, speed_range, dynamics, rng,
                   max_attempts=1000):
    """Truth trajectory by the reference's law (synthesis.py:95-121): start
    uniform in the interior, speed U[speed_min, speed_max], heading U[0, 2 pi),
    then the nearly-constant-velocity model; redrawn until it stays inside.
    Returns (frames + 1, 5): the state at k = 0 .. frames."""
    x_hi, y_hi = width - 1 - margin, height - 1 - margin
    if x_hi <= margin or y_hi <= margin:
        raise ConfigError("frame too small for the interior margin")
    noise = np.array([dynamics.sigma_pos, dynamics.sigma_pos, dynamics.sigma_vel,
                      dynamics.sigma_vel, dynamics.sigma_int])
    for _ in range(max_attempts):
        st = np.empty((frames + 1, 5))
        speed = rng.uniform(*speed_range)
        heading = rng.uniform(0.0, 2.0 * math.pi)
        st[0] = (rng.uniform(margin, x_hi), rng.uniform(margin, y_hi), speed * math.cos(heading),
                 speed * math.sin(heading), i0)
        for k in range(1, frames + 1):
            p = st[k - 1].copy()
            p[0] += p[2] * dynamics.dt
            p[1] += p[3] * dynamics.dt
            p += rng.normal(size=5) * noise
            p[4] = max(p[4], 0.0)
            st[k] = p
        if (st[:, 0].min() >= margin and st[:, 0].max() <= x_hi and st[:, 1].min() >= margin
                and st[:, 1].max() <= y_hi):
            return st
    raise ConfigError(f"no in-bounds trajectory found in {max_attempts} attempts")


def run_tracking_experiment(variants, n_particles, repetitions, scene=None, sigma_xi=10.0,
                            window_halfwidth=5, filter_dynamics=DynamicsParams(0.5, 0.1, 1.0),
                            truth_dynamics=DynamicsParams(0.05, 0.05, 0.0), i0=20.0,
                            speed_range=(0.3, 0.7), prior_sigma=2.0, seed=0,
                            experiment="gpu_tracking", progress=None):
    """Accuracy/runtime sweep (experiments.py:251-292) on the device.

    Every variant and N within a repetition runs on the same rendered
    sequence (paired comparisons). Degenerate weights are recorded as a
    failed run and do not abort the sweep."""
    scene = scene or syn.SceneConfig(PsfParams(1.5, 10.0), frames=20, width=128, height=128)
    specs = [parse_variant(v) for v in variants]
    ns = list(n_particles)
    if not ns or any(n < 1 for n in ns) or any(b <= a for a, b in zip(ns, ns[1:])):
        raise ConfigError("n_particles must be nonempty, >= 1 and strictly increasing")
    if repetitions < 1:
        raise ConfigError("repetitions must be >= 1")
    if sigma_xi <= 0:
        raise ConfigError("sigma_xi must be > 0")
    records = []
    for rep in range(repetitions):
        rng = np.random.default_rng(derive_seed(seed, "scene", experiment, rep))
        truth = generate_truth(scene.width, scene.height, scene.frames, window_halfwidth, i0,
                               speed_range, truth_dynamics, rng)
        frames = syn.render_sequence(truth[1:], scene,
                                     seed=derive_seed(seed, "noise", experiment, rep))
        init = InitSpec(StateVector(*truth[0]), "gauss", sigma=prior_sigma)
        for spec in specs:
            for n in ns:
                lik = SpotLikelihood(scene.psf, LikelihoodParams(sigma_xi, window_halfwidth))
                res = ResampleConfig(1.0, "systematic")
                rng_f = PhiloxRng(derive_seed(seed, "filter", spec.label, n, rep))
                if spec.is_pc:
                    grid = BinGrid.pixel_aligned(scene.width, scene.height, spec.cells_per_pixel)
                    cfg = PcFilterConfig(n, init, filter_dynamics, res, lik, grid=grid,
                                         placement=spec.placement)
                    track = pcsir_track
                else:
                    cfg = FilterConfig(n, init, filter_dynamics, res, lik)
                    track = sir_track
                torch.cuda.synchronize()
                start = time.perf_counter()
                try:
                    result = track(frames, cfg, rng_f)
                except DegenerateWeightsError:
                    records.append(RunRecord(experiment, spec.label, n, rep, float("nan"),
                                             time.perf_counter() - start, lik.evals, failed=True))
                    continue
                elapsed = time.perf_counter() - start
                d = result.positions - truth[1:, :2]
                rmse = float(np.sqrt(np.mean(np.sum(d ** 2, axis=1))))
                records.append(RunRecord(experiment, spec.label, n, rep, rmse, elapsed,
                                         result.likelihood_evals, trajectory=result.positions))
                if progress is not None:
                    progress(records[-1])
    return records


def run_tracking_on_scenes(scenes, variants, n_particles, psf, sigma_xi, window_halfwidth,
                           filter_dynamics=DynamicsParams(0.5, 0.5, 0.0), prior="point",
                           resampling=None, seed=0, experiment="small_object",
                           weighted_com=False, progress=None):
    """The reference's sweep (experiments.py:251-292) on given scenes: every
    variant and N of a repetition runs on the same frames (paired), with the
    reference harness's filter setup — prior parse_prior(prior, truth initial
    state), filter dynamics, ``ResampleConfig()`` (threshold 0.5, multinomial)
    unless ``resampling`` is given, weighted centre of mass optional — on the
    device filters. ``scenes``: iterable of dicts with ``frames`` (K, H, W),
    ``positions`` (K, 2) and ``init_state`` (5,) (e.g. the reference's own
    rendered scenes, tests/golden/experiments.npz). Wall time covers the
    filtering call only."""
    specs = [parse_variant(v) for v in variants]
    res = resampling if resampling is not None else ResampleConfig()
    records = []
    for rep, sc in enumerate(scenes):
        frames = torch.from_numpy(np.ascontiguousarray(np.asarray(sc["frames"], dtype=np.float32)))
        frames = frames.to(torch.device("cuda"))
        k, h, w = frames.shape
        center = StateVector(*np.asarray(sc["init_state"], dtype=np.float64))
        init = parse_prior(prior, center)
        truth_xy = np.asarray(sc["positions"], dtype=np.float64)
        for spec in specs:
            for n in n_particles:
                lik = SpotLikelihood(psf, LikelihoodParams(sigma_xi, window_halfwidth))
                if spec.is_pc:
                    grid = BinGrid.pixel_aligned(w, h, spec.cells_per_pixel)
                    cfg = PcFilterConfig(n, init, filter_dynamics, res, lik, grid=grid,
                                         placement=spec.placement, weighted_com=weighted_com)
                    track = pcsir_track
                else:
                    cfg = FilterConfig(n, init, filter_dynamics, res, lik)
                    track = sir_track
                rng_f = PhiloxRng(derive_seed(seed, "filter", spec.label, n, rep))
                torch.cuda.synchronize()
                start = time.perf_counter()
                try:
                    result = track(frames, cfg, rng_f)
                except DegenerateWeightsError:
                    records.append(RunRecord(experiment, spec.label, n, rep, float("nan"),
                                             time.perf_counter() - start, lik.evals, failed=True))
                    continue
                elapsed = time.perf_counter() - start
                d = result.positions - truth_xy
                rmse = float(np.sqrt(np.mean(np.sum(d ** 2, axis=1))))
                records.append(RunRecord(experiment, spec.label, n, rep, rmse, elapsed,
                                         result.likelihood_evals, trajectory=result.positions))
                if progress is not None:
                    progress(records[-1])
    return records


PSEUDO_PRIORS = ("uniform3x3", "uniform5x5", "gauss0.5", "gauss0.8")


def parse_prior(label, center: StateVector) -> InitSpec:
    """'point', 'uniform<w>[x<w>]' or 'gauss<s>' (experiments.py:73-90)."""
    token = label.strip().lower().replace("(", "").replace(")", "")
    try:
        if token == "point":
            return InitSpec(center, "point")
        if token.startswith("uniform"):
            return InitSpec(center, "uniform", width=float(token[7:].split("x")[0]))
        if token.startswith("gauss"):
            return InitSpec(center, "gauss", sigma=float(token[5:]))
    except ValueError:
        pass
    raise ConfigError(f"unknown prior {label!r}")


def pseudo_weight_once(pset: ParticleSet, frame, lik, spec: VariantSpec, grid=None,
                       weighted_com=False) -> ParticleSet:
    """One likelihood weighting of a particle cloud, no dynamics
    (experiments.py:295-310): SIR weights every particle; pcSIR bins,
    evaluates the dummies and broadcasts."""
    if not spec.is_pc:
        logw = _weight_update(pset, _evaluate_loglik(lik, pset.soa, frame))
    else:
        part = partition_device(pset.soa, grid)
        prior_w = pset.weights_f32().contiguous() if weighted_com else None
        dummies = dummy_states_device(pset.soa, grid, part, spec.placement, prior_w)
        logw = _weight_update(pset, _evaluate_loglik(lik, dummies, frame, cells=True), part.bin_of)
    _check_not_degenerate(logw)
    return ParticleSet.from_device(pset.soa, logw=logw, timestep=1)


def run_pseudo_tracking(variants, n_particles, repetitions, prior="uniform3x3", scene=None,
                        sigma_xi=10.0, window_halfwidth=5, i0=20.0, seed=0, weighted_com=False,
                        progress=None):
    """Single-frame convergence study (experiments.py:313-359) on the GPU.

    Per (N, repetition): a noise-free spot at a sub-pixel offset from the
    frame centre (all repetitions of an N rendered in one device call), a
    fresh cloud from the prior, weighted once through every variant; the
    record's error is |weighted-mean position - truth|."""
    scene = scene or syn.SceneConfig(PsfParams(1.5, 10.0), frames=1, width=64, height=64,
                                     noise=False)
    specs = [parse_variant(v) for v in variants]
    ns = list(n_particles)
    if not ns or any(n < 1 for n in ns) or repetitions < 1:
        raise ConfigError("n_particles must be nonempty and >= 1, repetitions >= 1")
    cx, cy = (scene.width - 1) / 2.0, (scene.height - 1) / 2.0
    parse_prior(prior, StateVector(cx, cy, 0.0, 0.0, i0))
    records = []
    for n in ns:
        offs = np.array([np.random.default_rng(derive_seed(seed, "pseudo", prior, n, r))
                         .uniform(-0.5, 0.5, size=2) for r in range(repetitions)])
        spots = np.stack([cx + offs[:, 0], cy + offs[:, 1], np.full(repetitions, i0)], axis=1)
        frames = syn.render_frames(spots, scene.width, scene.height, scene.psf, noise=False)
        for rep in range(repetitions):
            truth = StateVector(spots[rep, 0], spots[rep, 1], 0.0, 0.0, i0)
            frame = ImageFrame(frames[rep])
            base = init_particle_set(n, parse_prior(prior, truth),
                                     PhiloxRng(derive_seed(seed, "cloud", prior, n, rep)))
            for spec in specs:
                lik = SpotLikelihood(scene.psf, LikelihoodParams(sigma_xi, window_halfwidth))
                grid = (BinGrid.pixel_aligned(scene.width, scene.height, spec.cells_per_pixel)
                        if spec.is_pc else None)
                torch.cuda.synchronize()
                start = time.perf_counter()
                try:
                    w = normalize(pseudo_weight_once(base, frame, lik, spec, grid, weighted_com))
                    est = posterior_mean(w)
                except DegenerateWeightsError:
                    records.append(RunRecord("pseudo_tracking", spec.label, n, rep, float("nan"),
                                             time.perf_counter() - start, lik.evals, failed=True))
                    continue
                elapsed = time.perf_counter() - start
                err = float(np.hypot(est[0] - truth.x, est[1] - truth.y))
                records.append(RunRecord("pseudo_tracking", spec.label, n, rep, err, elapsed,
                                         lik.evals))
                if progress is not None:
                    progress(records[-1])
    return records


def _mean_std(values):
    if not values:
        return float("nan"), float("nan")
    mean = sum(values) / len(values)
    if len(values) == 1:
        return mean, 0.0
    return mean, math.sqrt(sum((v - mean) ** 2 for v in values) / (len(values) - 1))


def summarize(records) -> list:
    """Per-(variant, N) summary rows (reports.py:53-91): failed runs
    excluded; speedup_vs_sir = SIR mean time / variant mean time at equal N."""
    groups, order = {}, []
    for rec in records:
        key = (rec.variant, rec.n_particles)
        if key not in groups:
            groups[key] = []
            order.append(key)
        groups[key].append(rec)
    rows = []
    for variant, n in order:
        recs = [r for r in groups[(variant, n)] if not r.failed]
        rmse_mean, rmse_std = _mean_std([r.rmse for r in recs])
        if groups[(variant, n)][0].experiment == "pseudo_tracking":   # single-shot errors
            errs = [r.rmse for r in recs]
            rmse_mean = math.sqrt(sum(e * e for e in errs) / len(errs)) if errs else float("nan")
        t_mean, t_std = _mean_std([r.wall_time_s for r in recs])
        ev_mean, _ = _mean_std([r.lik_evals for r in recs])
        rows.append(SummaryRow(groups[(variant, n)][0].experiment, variant, n, rmse_mean, rmse_std,
                               t_mean, t_std, ev_mean, float("nan")))
    base = {r.n_particles: r.time_mean_s for r in rows if r.variant == "SIR"}
    for r in rows:
        if r.variant == "SIR":
            r.speedup_vs_sir = 1.0
        elif r.n_particles in base:
            r.speedup_vs_sir = base[r.n_particles] / r.time_mean_s
    return rows


def write_summary_csv(rows, path):
    """CSV with the reference's summary columns (reports.py:96-110)."""
    path = Path(path)
    path.parent.mkdir(parents=True, exist_ok=True)
    with open(path, "w") as f:
        f.write(",".join(SUMMARY_COLUMNS) + "\n")
        for r in rows:
            f.write(",".join(repr(getattr(r, c)) if isinstance(getattr(r, c), float)
                             else str(getattr(r, c)) for c in SUMMARY_COLUMNS) + "\n")
    return path


def likelihood_benchmark(repeats=5, seed=0, report=print):
    """Device likelihood operator on the reference's two micro-benchmark
    workloads (cli.py:191-213: a 512x512 Poisson(10) frame, 20000 9x9-window
    and 2000 65x65-window evaluations); returns {label: evals/s}."""
    rng = np.random.default_rng(seed)
    frame = rng.poisson(10.0, size=(512, 512)).astype(np.float64)
    out = {}
    for label, hw, n in (("small spot (9x9)", 4, 20000), ("large spot (65x65)", 32, 2000)):
        xs, ys = rng.uniform(40, 470, n), rng.uniform(40, 470, n)
        i0s = rng.uniform(5, 25, n)
        spot_window_ssd(frame, xs, ys, i0s, 1.16, 10.0, hw)   # warm-up / upload
        best = float("inf")
        for _ in range(repeats):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            spot_window_ssd(frame, xs, ys, i0s, 1.16, 10.0, hw)
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        out[label] = n / best
        report(f"{label:>18s} {'cuda':>9s}: {n / best:12.0f} evals/s")
    return out


# ---------------------------------------------------------------------------
# appendix bound study (experiments.py:362-388) on the device
# ---------------------------------------------------------------------------
BOUND_CELL_SIZES = (1.0, 0.5, 0.25, 0.125)
BOUND_DOMAINS = {
    "quadratic": (0.0, 4.0, 0.0, 4.0),
    "gaussian": (-4.0, 4.0, -4.0, 4.0),
    "sinsin": (0.0, 4.0, 0.0, 4.0),
}


def run_bounds_study(cell_sizes=BOUND_CELL_SIZES, fields=None) -> dict:
    """True mid-point approximation error versus both bounds:
    {field name: [(cell size, true error, rect bound, square bound)]} for
    uniform square partitions of each field's standard domain."""
    from .bounds import DomainPartition, builtin_fields, midpoint_error, rect_bound, square_bound
    fields = fields if fields is not None else builtin_fields()
    results = {}
    for name, fld in fields.items():
        domain = BOUND_DOMAINS[name]
        rows = []
        for l in cell_sizes:
            n_cols = int(round((domain[1] - domain[0]) / l))
            n_rows = int(round((domain[3] - domain[2]) / l))
            part = DomainPartition.uniform(domain, n_cols, n_rows)
            rows.append((l, midpoint_error(fld, part), rect_bound(fld, part),
                         square_bound(fld, l, domain)))
        results[name] = rows
    return results

