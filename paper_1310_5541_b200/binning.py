"""Piecewise-constant likelihood approximation over a spatial bin grid (pcSIR).

Mirrors ``pcsir.binning`` (binning.py:1-226). Particles are partitioned by
their (x, y) position into cells; each occupied cell gets one dummy state
(exact mean of its members, or the cell centre); the likelihood is evaluated
once per occupied cell and multiplies every member's weight.

Device paths: ``_partition`` / ``_dummy_states`` / ``pc_sis_step`` use the
general sort path (``pcs_partition``: CUB radix sort on 64-bit cell keys,
exact integer per-bin sums); ``pcsir_track`` runs the fused device loop
(dense bin window in HBM + shared-memory pre-aggregation, one CUDA graph per
frame) and falls back to the general driver only when the occupied-bin
window exceeds the fused capacity.
"""

import ctypes
import enum
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .filtering import (DegenerateWeightsError, FilterConfig, TrackResult, _check_not_degenerate,
                        _evaluate_loglik, _fused_ok, _track, _weight_update, fused_track)
from .rng import as_philox
from .state import I0, STATE_DIM, X, Y, ParticleSet, StateVector, propagate_array


class DummyPlacement(enum.Enum):
    """Where the per-cell representative state sits spatially (binning.py:21-25)."""

    CENTER_OF_MASS = "com"
    CELL_CENTER = "coc"


@dataclass(frozen=True)
class BinGrid:
    """Uniform rectangular cells tiling the tracking domain (binning.py:28-77)."""

    origin_x: float
    origin_y: float
    cell_width: float
    cell_height: float
    n_cols: int
    n_rows: int

    def __post_init__(self):
        if self.cell_width <= 0 or self.cell_height <= 0:
            raise ValueError("cell dimensions must be > 0")
        if self.n_cols < 1 or self.n_rows < 1:
            raise ValueError("grid extent must be >= 1 cell per axis")

    @classmethod
    def pixel_aligned(cls, width, height, cells_per_pixel=1):
        size = 1.0 / cells_per_pixel
        return cls(origin_x=-0.5, origin_y=-0.5, cell_width=size, cell_height=size,
                   n_cols=width * cells_per_pixel, n_rows=height * cells_per_pixel)

    def _axis(self, axis):
        return ((self.origin_x, self.cell_width, self.n_cols) if axis == 0
                else (self.origin_y, self.cell_height, self.n_rows))

    def cell_indices(self, xs, ys):
        """Column/row indices for coordinate arrays, clamped to the extent
        (host helper; the device path is pcs_common.cuh cell_axis)."""
        out = []
        for axis, v in ((0, xs), (1, ys)):
            o, size, n = self._axis(axis)
            k = np.floor((np.asarray(v) - o) / size)
            out.append(np.clip(k, 0, n - 1).astype(np.int64))
        return tuple(out)

    def cell_center(self, ix, iy):
        (ox, sx, _), (oy, sy, _) = self._axis(0), self._axis(1)
        return ox + (ix + 0.5) * sx, oy + (iy + 0.5) * sy

    def cell_bounds(self, ix, iy):
        (ox, sx, _), (oy, sy, _) = self._axis(0), self._axis(1)
        left, bottom = ox + ix * sx, oy + iy * sy
        return left, left + sx, bottom, bottom + sy

    def to_c(self):
        return _lib.PcsGrid(float(self.origin_x), float(self.origin_y), float(self.cell_width),
                            float(self.cell_height), int(self.n_cols), int(self.n_rows))


@dataclass
class BinOccupancy:
    """Sparse partition of particle indices by cell (binning.py:80-94)."""

    members: dict
    dummies: dict

    @property
    def n_occupied(self):
        return len(self.members)


@dataclass
class DevicePartition:
    """Device result of ``pcs_partition`` (binning.py:97-112 outputs, plus bin_of)."""

    flat: torch.Tensor      # (N,) uint64-as-int64 cell id per particle
    order: torch.Tensor     # (N,) int32 stable argsort
    bin_of: torch.Tensor    # (N,) int32 occupied-bin rank per particle
    unique: torch.Tensor    # (M,) cell ids ascending
    starts: torch.Tensor    # (M,) int64
    counts: torch.Tensor    # (M,) int64
    m: int


def partition_device(soa, grid: BinGrid) -> DevicePartition:
    n = soa.shape[1]
    dev = soa.device
    flat = torch.empty(n, dtype=torch.int64, device=dev)
    order = torch.empty(n, dtype=torch.int32, device=dev)
    bin_of = torch.empty(n, dtype=torch.int32, device=dev)
    unique = torch.empty(n, dtype=torch.int64, device=dev)
    starts = torch.empty(n, dtype=torch.int64, device=dev)
    counts = torch.empty(n, dtype=torch.int64, device=dev)
    m = ctypes.c_int64()
    g = grid.to_c()
    _lib.check(_lib.lib().pcs_partition(_lib.ctx(), _lib.ptr(soa), n, n, ctypes.byref(g),
                                        _lib.ptr(flat), _lib.ptr(order), _lib.ptr(bin_of),
                                        _lib.ptr(unique), _lib.ptr(starts), _lib.ptr(counts),
                                        ctypes.byref(m), _lib.stream()), "pcs_partition")
    mm = int(m.value)
    return DevicePartition(flat, order, bin_of, unique[:mm], starts[:mm], counts[:mm], mm)


def _soa_of(states):
    if isinstance(states, ParticleSet):
        return states.soa
    if isinstance(states, torch.Tensor) and states.is_cuda and states.shape[0] == STATE_DIM:
        return states.contiguous()
    arr = np.asarray(states, dtype=np.float64)
    return torch.from_numpy(np.ascontiguousarray(arr.T.astype(np.float32))).to(_lib.device())


def _partition(states, grid: BinGrid):
    """(flat, order, unique, starts, counts) as host int64 arrays (binning.py:97-112)."""
    p = partition_device(_soa_of(states), grid)
    u64 = lambda t: t.cpu().numpy().view(np.uint64).astype(np.int64)  # noqa: E731
    return (u64(p.flat), p.order.long().cpu().numpy(), u64(p.unique),
            p.starts.cpu().numpy(), p.counts.cpu().numpy())


def assign_bins(pset: ParticleSet, grid: BinGrid) -> BinOccupancy:
    """Partition the particles of a set by spatial cell (binning.py:115-126)."""
    _, order, unique, starts, counts = _partition(pset.soa, grid)
    ends = starts + counts
    members = {}
    for flat, lo, hi in zip(unique.tolist(), starts.tolist(), ends.tolist()):
        row, col = divmod(flat, grid.n_cols)
        members[(col, row)] = order[lo:hi]
    return BinOccupancy(members=members, dummies={})


def make_dummy(members, cell_bounds, placement: DummyPlacement, weights=None) -> StateVector:
    """Representative state for one cell's member states (binning.py:129-154),
    computed on the device (pcs_make_dummy) in float64 with the reference's
    summation orders: centre of mass = np.add.reduceat mean (single members
    reproduce themselves bit for bit), weighted by ``weights`` when given;
    cell centre puts x, y at the middle of ``cell_bounds``."""
    if len(members) == 0:
        raise ValueError("a dummy needs at least one member state")
    rows = np.atleast_2d(np.asarray(
        [m.as_array() if isinstance(m, StateVector) else m for m in members], dtype=np.float64))
    _lib.require_cuda()
    dev = _lib.device()
    r = torch.from_numpy(np.ascontiguousarray(rows)).to(dev)
    w = None
    if weights is not None:
        w = torch.from_numpy(np.ascontiguousarray(np.asarray(weights, dtype=np.float64))).to(dev)
        if w.numel() != r.shape[0]:
            raise ValueError("one weight per member is required")
    out = torch.empty(5, dtype=torch.float64, device=dev)
    pl = 1 if placement is DummyPlacement.CELL_CENTER else 0
    b = (ctypes.c_double * 4)(*[float(v) for v in cell_bounds])
    _lib.check(_lib.lib().pcs_make_dummy(_lib.ptr(r), r.shape[0], _lib.ptr(w), pl, b,
                                         _lib.ptr(out), _lib.stream()), "pcs_make_dummy")
    return StateVector.from_array(out.cpu().numpy())


def dummy_states_device(soa, grid, part: DevicePartition, placement, prior_w=None):
    """(5,M) float32 device dummies from the exact per-bin sums (binning.py:157-172)."""
    m = part.m
    d = torch.empty((STATE_DIM, m), dtype=torch.float32, device=soa.device)
    g = grid.to_c()
    pl = 1 if placement is DummyPlacement.CELL_CENTER else 0
    _lib.check(_lib.lib().pcs_dummies(_lib.ctx(), _lib.ptr(soa), soa.shape[1], soa.shape[1],
                                      _lib.ptr(part.order), _lib.ptr(part.bin_of),
                                      _lib.ptr(part.counts), _lib.ptr(part.unique), m,
                                      ctypes.byref(g), pl, _lib.ptr(prior_w), _lib.ptr(d), m,
                                      _lib.stream()), "pcs_dummies")
    return d


def _dummy_states(states, grid, order=None, unique=None, starts=None, counts=None,
                  placement=DummyPlacement.CENTER_OF_MASS, weights=None):
    """Representative state rows per occupied cell as host (M,5) float64 (binning.py:157-172).

    ``order/unique/starts/counts`` are accepted for signature compatibility;
    the partition is recomputed on the device from ``states``.
    """
    soa = _soa_of(states)
    part = partition_device(soa, grid)
    pw = None
    if weights is not None:
        w = np.empty(soa.shape[1], dtype=np.float32)
        order_h = part.order.long().cpu().numpy()
        w[order_h] = np.asarray(weights, dtype=np.float32)  # weights given in sorted order
        pw = torch.from_numpy(w).to(soa.device)
    d = dummy_states_device(soa, grid, part, placement, pw)
    return d.double().t().contiguous().cpu().numpy()


def pc_sis_step(pset: ParticleSet, frame, lik, dyn, grid: BinGrid, placement: DummyPlacement,
                rng, weighted_com=False, frame_id=None):
    """Propagate, bin, evaluate once per occupied cell, broadcast (binning.py:175-195).

    Returns (new ParticleSet, number of occupied cells).
    """
    states = propagate_array(pset.soa, dyn, rng, frame=frame_id)
    part = partition_device(states, grid)
    prior_w = None
    if weighted_com:
        prior_w = pset.weights_f32().contiguous()
    dummies = dummy_states_device(states, grid, part, placement, prior_w)
    cell_ll = _evaluate_loglik(lik, dummies, frame, cells=True)
    logw = _weight_update(pset, cell_ll, part.bin_of)
    _check_not_degenerate(logw)
    return ParticleSet.from_device(states, logw=logw, timestep=pset.timestep + 1), part.m


@dataclass(frozen=True)
class PcFilterConfig(FilterConfig):
    """Filter configuration plus the binning grid and dummy placement (binning.py:198-209)."""

    grid: BinGrid = None
    placement: DummyPlacement = DummyPlacement.CENTER_OF_MASS
    weighted_com: bool = False

    def __post_init__(self):
        super().__post_init__()
        if self.grid is None:
            raise ValueError("a bin grid is required")


def pcsir_track(frames, cfg: PcFilterConfig, rng, fused=None) -> TrackResult:
    """Piecewise-constant SIR (binning.py:212-226).

    With one particle per cell and centre-of-mass placement the trajectories
    match ``sir_track`` bit for bit under the same seed (exact integer
    per-bin sums make the dummies equal their single member).
    """
    prng = as_philox(rng)
    if fused is None:
        fused = _fused_ok(cfg)
    if fused:
        start = (prng.seed, prng.frame)
        try:
            pl = 1 if cfg.placement is DummyPlacement.CELL_CENTER else 0
            return fused_track(frames, cfg, prng, method=1, grid=cfg.grid, placement=pl)
        except _lib.CapacityError:
            prng.seed, prng.frame = start

    def step(pset, frame, rng_, frame_id):
        new_set, _ = pc_sis_step(pset, frame, cfg.likelihood, cfg.dynamics, cfg.grid,
                                 cfg.placement, rng_, weighted_com=cfg.weighted_com,
                                 frame_id=frame_id)
        return new_set

    return _track(frames, cfg, prng, step)
