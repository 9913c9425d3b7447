"""State vectors, device particle sets and nearly-constant-velocity dynamics.

Mirrors the reference ``pcsir.state`` API (state.py:1-175) with the particle
set held on the GPU as float32 structure-of-arrays ``soa[c, i]``
(c in x, y, vx, vy, I0 — state.py:16). Weights are held in one of three
forms: uniform (all 1/N, nothing stored), normalised float32 ``w`` (after
``normalize``), or unnormalised float64 log-weights ``logw`` (after a step,
before ``normalize``). ``states`` / ``weights`` return host float64 copies
so reference-style code keeps working.
"""

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .rng import as_philox

X, Y, VX, VY, I0 = range(5)
STATE_DIM = 5


@dataclass(frozen=True)
class StateVector:
    """Single object state: position, velocity, peak intensity (state.py:20-40)."""

    x: float
    y: float
    vx: float
    vy: float
    intensity: float

    def __post_init__(self):
        if self.intensity < 0:
            raise ValueError("intensity must be >= 0")

    def as_array(self):
        return np.array([self.x, self.y, self.vx, self.vy, self.intensity])

    @classmethod
    def from_array(cls, row):
        return cls(float(row[X]), float(row[Y]), float(row[VX]), float(row[VY]), float(row[I0]))


@dataclass(frozen=True)
class Particle:
    """A weighted state sample (state.py:43-52)."""

    state: StateVector
    weight: float

    def __post_init__(self):
        if not np.isfinite(self.weight) or self.weight < 0:
            raise ValueError("weight must be finite and >= 0")


def _to_soa(states):
    """(N,5) array-like or (5,N) device tensor -> contiguous (5,N) float32 CUDA tensor."""
    dev = _lib.device()
    if isinstance(states, torch.Tensor) and states.is_cuda and states.dim() == 2 \
            and states.shape[0] == STATE_DIM and states.dtype == torch.float32:
        return states.contiguous()
    arr = np.asarray(states, dtype=np.float64)
    if arr.ndim != 2 or arr.shape[1] != STATE_DIM:
        raise ValueError("states must have shape (N, 5)")
    host = np.ascontiguousarray(arr.T.astype(np.float32))
    return torch.from_numpy(host).to(dev)


class ParticleSet:
    """N weighted state samples on the GPU (state.py:55-88).

    ``ParticleSet(states, weights, timestep)`` accepts host (N,5) states and
    (N,) weights like the reference; use :meth:`from_device` to wrap device
    buffers without a copy.
    """

    def __init__(self, states, weights=None, timestep=0):
        self.soa = _to_soa(states)
        n = self.soa.shape[1]
        if n < 1:
            raise ValueError("a particle set needs at least one particle")
        self.timestep = int(timestep)
        self.w = None        # normalised float32 weights
        self.logw = None     # unnormalised float64 log weights
        self.uniform = False
        if weights is None:
            self.uniform = True
        else:
            wt = np.asarray(weights, dtype=np.float64) if not isinstance(weights, torch.Tensor) \
                else weights.detach().double().cpu().numpy()
            if wt.shape != (n,):
                raise ValueError("weights must have shape (N,)")
            if np.all(wt == 1.0 / n):
                self.uniform = True
                return
            with np.errstate(divide="ignore"):
                self.logw = torch.from_numpy(np.log(wt)).to(self.soa.device)

    @classmethod
    def from_device(cls, soa, *, w=None, logw=None, uniform=False, timestep=0):
        obj = cls.__new__(cls)
        obj.soa = soa.contiguous()
        obj.timestep = int(timestep)
        obj.w = w
        obj.logw = logw
        obj.uniform = bool(uniform)
        if sum(x is not None for x in (w, logw)) + int(bool(uniform)) != 1:
            raise ValueError("exactly one weight form is required")
        return obj

    def __len__(self):
        return self.soa.shape[1]

    @property
    def n(self):
        return self.soa.shape[1]

    @property
    def states(self):
        """Host (N,5) float64 copy of the states."""
        return self.soa.double().t().contiguous().cpu().numpy()

    @property
    def weights(self):
        """Host (N,) float64 copy of the weights in the reference's linear domain."""
        if self.w is not None:
            return self.w.double().cpu().numpy()
        if self.uniform:
            return np.full(self.n, 1.0 / self.n)
        return torch.exp(self.logw).cpu().numpy()

    def weights_f32(self):
        """Device float32 weights (normalised form, uniform 1/N, or exp(logw))."""
        if self.w is not None:
            return self.w
        if self.uniform:
            return torch.full((self.n,), 1.0 / self.n, dtype=torch.float32, device=self.soa.device)
        return torch.exp(self.logw).float()

    def particle(self, i) -> Particle:
        return Particle(StateVector.from_array(self.states[i]), float(self.weights[i]))

    def copy(self):
        return ParticleSet.from_device(
            self.soa.clone(), w=None if self.w is None else self.w.clone(),
            logw=None if self.logw is None else self.logw.clone(), uniform=self.uniform,
            timestep=self.timestep)


@dataclass(frozen=True)
class DynamicsParams:
    """Process-noise magnitudes of the nearly-constant-velocity model (state.py:91-112)."""

    sigma_pos: float = 0.5
    sigma_vel: float = 0.5
    sigma_int: float = 0.0
    dt: float = 1.0

    def __post_init__(self):
        if min(self.sigma_pos, self.sigma_vel, self.sigma_int) < 0:
            raise ValueError("noise magnitudes must be >= 0")
        if self.dt <= 0:
            raise ValueError("dt must be > 0")

    def noise_scale(self):
        return np.array([self.sigma_pos, self.sigma_pos, self.sigma_vel, self.sigma_vel,
                         self.sigma_int])

    def to_c(self):
        return _lib.PcsDynamics(self.sigma_pos, self.sigma_vel, self.sigma_int, self.dt)


def propagate_array(states, params: DynamicsParams, rng, ancestors=None, frame=None):
    """Nearly-constant-velocity step on the GPU (state.py:115-127).

    ``states`` is a (5,N) device tensor or a host (N,5) array; returns a new
    (5,N) float32 device tensor. Consumes one Philox frame of N*5 normals
    (always, independent of which sigmas are zero, as state.py:118-119).
    ``ancestors`` fuses the resampling gather (filtering.py:107).
    """
    soa = _to_soa(states)
    n = soa.shape[1]
    if hasattr(rng, "replay_normals"):  # recorded draws (rng.ReplayNormals)
        return propagate_with_normals(soa, params, rng.replay_normals(n), ancestors)
    prng = as_philox(rng)
    f = prng.next_frame() if frame is None else frame
    out = torch.empty_like(soa)
    dyn = params.to_c()
    _lib.check(_lib.lib().pcs_propagate(
        _lib.ptr(soa), _lib.ptr(out), n, n, _lib.ptr(ancestors), ctypes.byref(dyn),
        prng.seed, f & 0xFFFFFFFF, 0, _lib.stream()), "pcs_propagate")
    return out


def propagate_with_normals(states, params: DynamicsParams, normals, ancestors=None):
    """Replay form of :func:`propagate_array`: the (5,N) standard normals are
    given (``pcs_propagate_given``) — runs the device arithmetic on recorded
    ``rng.normal(size=(N,5))`` draws for parity checks."""
    soa = _to_soa(states)
    n = soa.shape[1]
    z = normals if isinstance(normals, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(np.asarray(normals, dtype=np.float32)))
    z = z.to(soa.device, dtype=torch.float32).contiguous()
    if z.shape != (STATE_DIM, n):
        raise ValueError("normals must have shape (5, N)")
    out = torch.empty_like(soa)
    dyn = params.to_c()
    _lib.check(_lib.lib().pcs_propagate_given(
        _lib.ptr(soa), _lib.ptr(out), n, n, _lib.ptr(ancestors), ctypes.byref(dyn), _lib.ptr(z), n,
        _lib.stream()), "pcs_propagate_given")
    return out


def device_normals(seed, frame, n, offset=0):
    """The (5,N) float32 normals pcs_propagate draws at (seed, frame) (replay)."""
    out = torch.empty((STATE_DIM, n), dtype=torch.float32, device=_lib.device())
    _lib.check(_lib.lib().pcs_philox_normals(seed, frame & 0xFFFFFFFF, offset, n, _lib.ptr(out), n,
                                             _lib.stream()), "pcs_philox_normals")
    return out


def propagate(state: StateVector, params: DynamicsParams, rng) -> StateVector:
    """One step of a single state (state.py:130-137)."""
    out = propagate_array(state.as_array()[None, :], params, rng)
    return StateVector.from_array(out.double().cpu().numpy()[:, 0])


@dataclass(frozen=True)
class InitSpec:
    """How to draw the initial particle cloud around a centre state (state.py:140-161)."""

    center: StateVector
    mode: str = "point"
    width: float = 0.0
    sigma: float = 0.0

    def __post_init__(self):
        if self.mode not in ("point", "uniform", "gauss"):
            raise ValueError(f"unknown init mode {self.mode!r}")
        if self.mode == "uniform" and self.width <= 0:
            raise ValueError("uniform init needs width > 0")
        if self.mode == "gauss" and self.sigma <= 0:
            raise ValueError("gauss init needs sigma > 0")

    def to_c(self):
        c = _lib.PcsInit()
        for k, v in enumerate(self.center.as_array()):
            c.center[k] = float(v)
        c.mode = {"point": 0, "uniform": 1, "gauss": 2}[self.mode]
        c.width = float(self.width)
        c.sigma = float(self.sigma)
        return c


def init_particle_set(n, init: InitSpec, rng) -> ParticleSet:
    """Draw N particles per the init spec, all with weight 1/N (state.py:164-175)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    prng = as_philox(rng)
    dev = _lib.device()
    soa = torch.empty((STATE_DIM, n), dtype=torch.float32, device=dev)
    spec = init.to_c()
    _lib.check(_lib.lib().pcs_init_particles(ctypes.byref(spec), prng.seed, 0, n, _lib.ptr(soa), n,
                                             _lib.stream()), "pcs_init_particles")
    return ParticleSet.from_device(soa, uniform=True, timestep=0)
