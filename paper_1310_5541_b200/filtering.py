"""Sequential importance resampling on the GPU: weight updates, normalisation,
ESS, resampling and the frame-by-frame tracking driver.

Mirrors ``pcsir.filtering`` (filtering.py:1-182). Two drivers share one set
of canonical device arithmetic:

* the fused device loop (``pcs_track``: one captured CUDA graph per frame, no
  host synchronisation) for the built-in likelihoods, systematic or
  multinomial resampling at any ESS threshold;
* the general step-by-step driver (``_track``) for duck-typed likelihoods,
  grids whose occupied-bin window exceeds the fused capacity, and on request
  (``fused=False``).

Both produce identical estimates / ESS / resampling decisions.
"""

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .imaging import ImageFrame, _DeviceLikelihood
from .rng import PhiloxRng, as_philox
from .state import (DynamicsParams, InitSpec, ParticleSet, StateVector, init_particle_set,
                    propagate_array)


class DegenerateWeightsError(RuntimeError):
    """All particle weights vanished; the posterior approximation is gone (filtering.py:20-25)."""

    def __init__(self, message, frame_index=None):
        super().__init__(message)
        self.frame_index = frame_index


@dataclass(frozen=True)
class ResampleConfig:
    """When and how to resample (filtering.py:28-45)."""

    threshold_fraction: float = 0.5
    scheme: str = "multinomial"

    def __post_init__(self):
        if not 0.0 < self.threshold_fraction <= 1.0:
            raise ValueError("threshold_fraction must be in (0, 1]")
        if self.scheme not in ("multinomial", "systematic"):
            raise ValueError(f"unknown resampling scheme {self.scheme!r}")


def _evaluate_loglik(lik, soa, frame, cells=False):
    """Device log-likelihood per state column (filtering.py:48-59).

    Built-in likelihoods evaluate on the GPU in float32. A duck-typed object
    with ``.batch(states, frame)`` (the reference's test doubles) is called on
    a host float64 copy — conformance only, never the benchmarked path.
    """
    if isinstance(lik, _DeviceLikelihood):
        return lik.loglik(soa, frame, cells=cells)
    host_states = soa.double().t().contiguous().cpu().numpy()
    batch = getattr(lik, "batch", None)
    if batch is not None:
        values = np.asarray(batch(host_states, frame), dtype=np.float64)
    else:
        values = np.array([lik(StateVector.from_array(s), frame) for s in host_states])
    if values.shape != (host_states.shape[0],):
        raise ValueError("likelihood must return one value per particle")
    if not np.all(np.isfinite(values)) or np.any(values < 0):
        raise ValueError("likelihood values must be finite and >= 0")
    with np.errstate(divide="ignore"):
        ll = np.log(values)
    # keep float64 precision for host doubles: returned as float64 log-lik
    return torch.from_numpy(ll).to(soa.device)


def _weight_update(pset, ll, bin_of=None):
    """log w_new = log(w_prev) + ll[bin_of] in float64 (filtering.py:69, binning.py:190-192)."""
    n = pset.n
    dev = pset.soa.device
    ll = ll.to(dtype=torch.float64).contiguous()
    logw = torch.empty(n, dtype=torch.float64, device=dev)
    _lib.check(_lib.lib().pcs_weight_update(
        _lib.ptr(pset.w), _lib.ptr(pset.logw), _lib.ptr(ll), _lib.ptr(bin_of), n,
        _lib.ptr(logw), _lib.stream()), "pcs_weight_update")
    return logw


def _check_not_degenerate(logw):
    if not bool(torch.any(logw > -float("inf"))):
        raise DegenerateWeightsError("all importance weights vanished")


def sis_step(pset: ParticleSet, frame: ImageFrame, lik, dyn: DynamicsParams, rng,
             frame_id=None) -> ParticleSet:
    """Propagate every particle, then scale its weight by its likelihood (filtering.py:62-72)."""
    states = propagate_array(pset.soa, dyn, rng, frame=frame_id)
    ll = _evaluate_loglik(lik, states, frame)
    logw = _weight_update(pset, ll)
    _check_not_degenerate(logw)
    return ParticleSet.from_device(states, logw=logw, timestep=pset.timestep + 1)


def normalize(pset: ParticleSet) -> ParticleSet:
    """Rescale weights to sum to one (filtering.py:75-85), in the log domain on the GPU."""
    n = pset.n
    dev = pset.soa.device
    if pset.logw is not None:
        logw = pset.logw.contiguous()
    elif pset.uniform:
        logw = torch.zeros(n, dtype=torch.float64, device=dev)
    else:
        logw = torch.log(pset.w.double())
    w = torch.empty(n, dtype=torch.float32, device=dev)
    mx = ctypes.c_double()
    nm = ctypes.c_double()
    deg = ctypes.c_int32()
    _lib.check(_lib.lib().pcs_normalize(_lib.ctx(), _lib.ptr(logw), n, _lib.ptr(w),
                                        ctypes.byref(mx), ctypes.byref(nm), ctypes.byref(deg),
                                        _lib.stream()), "pcs_normalize")
    if deg.value:
        raise DegenerateWeightsError("weight sum is zero, cannot normalize")
    return ParticleSet.from_device(pset.soa, w=w, timestep=pset.timestep)


def _estimate_ess(pset):
    w = pset.weights_f32().contiguous()
    est = (ctypes.c_double * 5)()
    ess = ctypes.c_double()
    _lib.check(_lib.lib().pcs_estimate_ess(_lib.ctx(), _lib.ptr(pset.soa), pset.n, _lib.ptr(w),
                                           pset.n, est, ctypes.byref(ess), _lib.stream()),
               "pcs_estimate_ess")
    return np.array(est[:]), float(ess.value)


def effective_sample_size(pset: ParticleSet) -> float:
    """1 / sum(w^2) (filtering.py:88-90), exact fixed-point sum on the GPU."""
    if pset.logw is not None:
        w = torch.exp(pset.logw)
        return 1.0 / float(torch.sum(w * w))
    return _estimate_ess(pset)[1]


def posterior_mean(pset: ParticleSet) -> np.ndarray:
    """Weighted mean state under normalised weights (filtering.py:112-114)."""
    if pset.logw is not None:
        w = torch.exp(pset.logw)
        return (pset.soa.double() @ w).cpu().numpy()
    return _estimate_ess(pset)[0]


def _ancestors(pset, cfg: ResampleConfig, prng: PhiloxRng, frame=None):
    n = pset.n
    w = pset.weights_f32().contiguous()
    anc = torch.empty(n, dtype=torch.int32, device=pset.soa.device)
    if cfg.scheme == "systematic":
        u = prng.resample_u(frame)
        _lib.check(_lib.lib().pcs_resample_systematic(_lib.ctx(), _lib.ptr(w), n, u,
                                                      _lib.ptr(anc), _lib.stream()),
                   "pcs_resample_systematic")
    else:
        f = prng.multinomial_frame() if frame is None else frame
        pts = torch.empty(n, dtype=torch.float64, device=pset.soa.device)
        _lib.check(_lib.lib().pcs_philox_multinomial_points(prng.seed, f & 0xFFFFFFFF, n,
                                                            _lib.ptr(pts), _lib.stream()),
                   "pcs_philox_multinomial_points")
        _lib.check(_lib.lib().pcs_resample_multinomial(_lib.ctx(), _lib.ptr(w), n, _lib.ptr(pts),
                                                       _lib.ptr(anc), _lib.stream()),
                   "pcs_resample_multinomial")
    return anc


def resample_indices(pset: ParticleSet, cfg: ResampleConfig, rng, frame=None):
    """Ancestor indices (filtering.py:93-100) as a device int32 tensor."""
    return _ancestors(pset, cfg, as_philox(rng), frame)


def resample(pset: ParticleSet, cfg: ResampleConfig, rng, frame=None) -> ParticleSet:
    """Draw N copies with probability equal to the weights, reset weights to 1/N
    (filtering.py:103-109)."""
    anc = _ancestors(pset, cfg, as_philox(rng), frame)
    out = torch.empty_like(pset.soa)
    _lib.check(_lib.lib().pcs_gather(_lib.ptr(pset.soa), _lib.ptr(out), pset.n, pset.n,
                                     _lib.ptr(anc), _lib.stream()), "pcs_gather")
    return ParticleSet.from_device(out, uniform=True, timestep=pset.timestep)


@dataclass(frozen=True)
class FilterConfig:
    """Everything a tracking run needs besides the frames and the RNG (filtering.py:117-131)."""

    n_particles: int
    init: InitSpec
    dynamics: DynamicsParams = DynamicsParams()
    resampling: ResampleConfig = ResampleConfig()
    likelihood: object = None

    def __post_init__(self):
        if self.n_particles < 1:
            raise ValueError("n_particles must be >= 1")
        if self.likelihood is None:
            raise ValueError("a likelihood evaluator is required")


@dataclass
class TrackResult:
    """Per-frame posterior-mean estimates plus run diagnostics (filtering.py:134-145)."""

    estimates: np.ndarray          # (K, 5) weighted means, pre-resampling
    ess: np.ndarray                # (K,) effective sample size per frame
    resampled: np.ndarray          # (K,) bool, resampled after this frame
    likelihood_evals: int          # total likelihood evaluations
    path: str = "general"          # "fused" (device loop) or "general"

    @property
    def positions(self):
        return self.estimates[:, :2]


def _all_equal(w):
    return bool(torch.all(w == w[0]))


def _track(frames, cfg: FilterConfig, rng, step_fn):
    """General driver: step -> normalize -> estimate -> conditional resample
    (filtering.py:148-173). Frame k propagates with Philox frame id k and
    resamples with u(seed, k), exactly as the fused device loop."""
    if len(frames) < 1:
        raise ValueError("need at least one frame")
    prng = as_philox(rng)
    frame0 = prng.frame
    evals_before = getattr(cfg.likelihood, "evals", 0)
    pset = init_particle_set(cfg.n_particles, cfg.init, prng)
    threshold = cfg.resampling.threshold_fraction * cfg.n_particles
    estimates = np.empty((len(frames), 5))
    ess_log = np.empty(len(frames))
    resampled = np.zeros(len(frames), dtype=bool)
    for k, frame in enumerate(frames):
        if not isinstance(frame, ImageFrame):   # rows of a (K,H,W) array / tensor
            frame = ImageFrame(frame)
        try:
            pset = step_fn(pset, frame, prng, frame0 + k)
            pset = normalize(pset)
        except DegenerateWeightsError as err:
            raise DegenerateWeightsError(str(err), frame_index=k) from None
        estimates[k], ess_log[k] = _estimate_ess(pset)
        if ess_log[k] < threshold:
            pset = resample(pset, cfg.resampling, prng, frame=frame0 + k)
            resampled[k] = True
        elif _all_equal(pset.w):
            pset = ParticleSet.from_device(pset.soa, uniform=True, timestep=pset.timestep)
    prng.frame = frame0 + len(frames)
    evals = getattr(cfg.likelihood, "evals", 0) - evals_before
    return TrackResult(estimates, ess_log, resampled, evals, "general")


def _frames_to_device(frames):
    """One (K,H,W) float32 device tensor of the frames. Accepts a list of
    ImageFrame / 2D arrays, a (K,H,W) array, or a (K,H,W) torch tensor (a
    pinned float32 host tensor is copied asynchronously on the current
    stream, which the filter kernels run on)."""
    if isinstance(frames, torch.Tensor):
        t = frames if frames.dtype == torch.float32 else frames.float()
        t = t.contiguous()
        if t.is_cuda:
            return t
        return t.to(_lib.device(), non_blocking=t.is_pinned())
    if isinstance(frames, np.ndarray) and frames.ndim == 3:
        host = np.ascontiguousarray(frames, dtype=np.float32)
    else:
        host = np.stack([f.pixels if isinstance(f, ImageFrame) else np.asarray(f) for f in frames],
                        dtype=np.float32)
    t = torch.from_numpy(host)
    if torch.cuda.is_available():
        t = t.pin_memory()
    return t.to(_lib.device(), non_blocking=True)


def fused_track(frames, cfg: FilterConfig, rng, method, grid=None, placement=0, use_graph=True):
    """Run the whole filter on the device (``pcs_track``); returns TrackResult
    or raises CapacityError when the general path is needed."""
    prng = as_philox(rng)
    frame0 = prng.frame
    # a pinned host tensor of >= 8 MB is uploaded in up to 4 chunks on a side
    # stream, each chunk's frames filtered as soon as it has arrived
    pipelined = (isinstance(frames, torch.Tensor) and not frames.is_cuda and frames.dim() == 3
                 and frames.dtype == torch.float32 and frames.is_pinned() and frames.shape[0] >= 2
                 and frames.numel() * 4 >= (8 << 20))
    if pipelined:
        host = frames.contiguous()
        dev_frames = torch.empty(host.shape, dtype=torch.float32, device=_lib.device())
        nch = min(4, host.shape[0])
        bounds = np.linspace(0, host.shape[0], nch + 1).astype(int)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())   # dev_frames allocated
        arrived = []
        with torch.cuda.stream(side):
            for a, b in zip(bounds[:-1], bounds[1:]):
                dev_frames[a:b].copy_(host[a:b], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(side)
                arrived.append(ev)
        # the side stream writes dev_frames: keep its memory until those copies
        # are done even if the filter raises before waiting on them
        dev_frames.record_stream(side)
    else:
        dev_frames = _frames_to_device(frames)
    k, h, w = dev_frames.shape
    lik = cfg.likelihood
    c = _lib.PcsTrackCfg()
    c.method = method
    c.placement = placement
    c.n_particles = cfg.n_particles
    c.init = cfg.init.to_c()
    c.dyn = cfg.dynamics.to_c()
    c.spot = lik.spot_c(cells=(method == 1))
    if grid is not None:
        c.grid = grid.to_c()
    c.seed = prng.seed
    c.frame0 = frame0
    c.use_graph = 1 if use_graph else 0
    c.threshold_fraction = cfg.resampling.threshold_fraction
    c.scheme = 1 if cfg.resampling.scheme == "multinomial" else 0
    c.weighted_com = 1 if (method == 1 and getattr(cfg, "weighted_com", False)) else 0
    dev = dev_frames.device
    est = torch.empty((k, 5), dtype=torch.float64, device=dev)
    ess = torch.empty(k, dtype=torch.float64, device=dev)
    res = torch.empty(k, dtype=torch.uint8, device=dev)
    occ = torch.empty(k, dtype=torch.int64, device=dev)
    out = _lib.PcsTrackResult()
    if pipelined:
        L, ctx, st = _lib.lib(), _lib.ctx(), _lib.stream()
        _lib.check(L.pcs_track_begin(ctx, ctypes.byref(c), h, w, st), "pcs_track_begin")
        for (a, b), ev in zip(zip(bounds[:-1], bounds[1:]), arrived):
            torch.cuda.current_stream().wait_event(ev)
            rc = L.pcs_track_steps(ctx, _lib.ptr(dev_frames[a:]), int(a), int(b), _lib.ptr(est[a:]),
                                   _lib.ptr(ess[a:]), _lib.ptr(res[a:]), _lib.ptr(occ[a:]), st)
            if rc:
                L.pcs_track_end(ctx, ctypes.byref(out), st)
                _lib.check(rc, "pcs_track_steps")
        _lib.check(L.pcs_track_end(ctx, ctypes.byref(out), st), "pcs_track")
    else:
        rc = _lib.lib().pcs_track(_lib.ctx(), ctypes.byref(c), _lib.ptr(dev_frames), k, h, w,
                                  _lib.ptr(est), _lib.ptr(ess), _lib.ptr(res), _lib.ptr(occ),
                                  ctypes.byref(out), _lib.stream())
        _lib.check(rc, "pcs_track")
    if out.flags & _lib.FLAG_NONFINITE:
        raise ValueError("likelihood values must be finite and >= 0")
    if out.flags & _lib.FLAG_DEGENERATE:
        raise DegenerateWeightsError("all importance weights vanished",
                                     frame_index=int(out.first_bad_frame))
    if out.flags & _lib.FLAG_RANGE:
        raise ValueError("particle state beyond the exact fixed-point range (|v| >= 2^24)")
    prng.frame = frame0 + k
    lik.evals += int(out.likelihood_evals)
    return TrackResult(est.cpu().numpy(), ess.cpu().numpy(), res.cpu().numpy().astype(bool),
                       int(out.likelihood_evals), "fused")


def _fused_ok(cfg):
    """The fused pcSIR loop: device likelihood, systematic or multinomial
    resampling, any ESS threshold (frames whose particles carry prior weights
    finish per particle on the device)."""
    r = cfg.resampling
    return (isinstance(cfg.likelihood, _DeviceLikelihood)
            and r.scheme in ("systematic", "multinomial") and cfg.n_particles < 2 ** 31 - 1)


def _fused_sir_ok(cfg):
    """The fused SIR loop also runs ESS-threshold resampling (threshold < 1):
    per-particle prior weights stay on the device between frames."""
    r = cfg.resampling
    return (isinstance(cfg.likelihood, _DeviceLikelihood)
            and r.scheme in ("systematic", "multinomial") and cfg.n_particles < 2 ** 31 - 1)


def sir_track(frames, cfg: FilterConfig, rng, fused=None) -> TrackResult:
    """Classical SIR: one likelihood evaluation per particle per frame (filtering.py:176-182)."""
    prng = as_philox(rng)
    if fused is None:
        fused = _fused_sir_ok(cfg)
    if fused:
        start = (prng.seed, prng.frame)
        try:
            return fused_track(frames, cfg, prng, method=0)
        except _lib.CapacityError:
            prng.seed, prng.frame = start

    def step(pset, frame, rng_, frame_id):
        return sis_step(pset, frame, cfg.likelihood, cfg.dynamics, rng_, frame_id=frame_id)

    return _track(frames, cfg, prng, step)
