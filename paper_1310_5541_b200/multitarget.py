"""Batched multi-target pcSIR (BASELINE config 4; new — the reference runs
one filter per spot, ``experiments.py:251-292`` loops targets /
repetitions serially).

``multi_pcsir_track`` runs T independent pcSIR filters over the same frame
sequence in one kernel launch per frame (one CTA per target, pcs_mt_*), with
the configuration's ResampleConfig (ESS threshold, systematic or multinomial;
filtering.py:38-39,96-100,169-171).
Target t uses the RNG key ``seed + t * 0x9E3779B97F4A7C15`` so it is exactly
``pcsir_track(frames, cfg_t, PhiloxRng(seed_t))`` with ``cfg_t`` centred on
target t. Across GPUs the targets are partitioned ([r*T/P, (r+1)*T/P) on rank
r) with no communication; ``gather_results`` optionally collects them.
"""

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

KEY_STEP = 0x9E3779B97F4A7C15


def target_seed(seed, t):
    return (seed + t * KEY_STEP) % (1 << 64)


def target_range(n_targets, rank, world):
    """Contiguous block of targets owned by ``rank`` (balanced, deterministic)."""
    base, extra = divmod(n_targets, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


@dataclass
class MultiTrackResult:
    estimates: np.ndarray      # (T, K, 5)
    ess: np.ndarray            # (T, K)
    resampled: np.ndarray      # (T, K)
    occupied: np.ndarray       # (T, K) likelihood evaluations per frame
    flags: np.ndarray          # (T,) PCS_FLAG_* per target
    likelihood_evals: np.ndarray  # (T,)


class MultiTargetTracker:
    """Device state of T filters; step() advances all of them by one frame."""

    def __init__(self, cfg, centers, seed, n_frames, height, width, target_offset=0):
        r = cfg.resampling
        if getattr(cfg, "weighted_com", False):
            raise ValueError("the multi-target kernel places dummies at the unweighted centre "
                             "of mass; run pcsir_track per target for weighted_com=True")
        centers = np.ascontiguousarray(np.asarray(centers, dtype=np.float64).reshape(-1, 5))
        self.T = centers.shape[0]
        self.K = n_frames
        c = _lib.PcsTrackCfg()
        c.method = 1
        c.placement = 1 if cfg.placement.value == "coc" else 0
        c.n_particles = cfg.n_particles
        c.init = cfg.init.to_c()
        c.dyn = cfg.dynamics.to_c()
        c.spot = cfg.likelihood.spot_c(cells=True)
        c.grid = cfg.grid.to_c()
        c.threshold_fraction = r.threshold_fraction      # filtering.py:169-171
        c.scheme = 1 if r.scheme == "multinomial" else 0  # filtering.py:96-100
        c.seed = seed % (1 << 64)
        c.frame0 = 0
        c.use_graph = 0
        self._cfg = c
        self._centers = centers
        _lib.check(_lib.lib().pcs_mt_begin(_lib.ctx(), ctypes.byref(c), self.T,
                                           centers.ctypes.data_as(ctypes.c_void_p),
                                           target_offset, n_frames, height, width, _lib.stream()),
                   "pcs_mt_begin")
        self.k = 0

    def step(self, frame):
        _lib.check(_lib.lib().pcs_mt_step(_lib.ctx(), _lib.ptr(frame), self.k, _lib.stream()),
                   "pcs_mt_step")
        self.k += 1

    def results(self):
        T, K = self.T, self.K
        est = np.empty((T, K, 5))
        ess = np.empty((T, K))
        res = np.empty((T, K), dtype=np.uint8)
        occ = np.empty((T, K), dtype=np.int64)
        flags = np.empty(T, dtype=np.uint32)
        evals = np.empty(T, dtype=np.int64)
        p = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        _lib.check(_lib.lib().pcs_mt_results(_lib.ctx(), p(est), p(ess), p(res), p(occ), p(flags),
                                             p(evals), _lib.stream()), "pcs_mt_results")
        return MultiTrackResult(est, ess, res.astype(bool), occ, flags, evals)


def multi_pcsir_track(frames, cfg, centers, seed, target_offset=0):
    """T independent pcSIR filters (config 4) on the device; frames (K,H,W)."""
    t = frames if isinstance(frames, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(np.asarray(frames, dtype=np.float32)))
    t = (t if t.dtype == torch.float32 else t.float()).contiguous()
    dev_frames = t if t.is_cuda else t.to(_lib.device(), non_blocking=t.is_pinned())
    k, h, w = dev_frames.shape
    tr = MultiTargetTracker(cfg, centers, seed, k, h, w, target_offset)
    for f in range(k):
        tr.step(dev_frames[f])
    r = tr.results()
    bad = r.flags & (_lib.FLAG_NONFINITE | _lib.FLAG_DEGENERATE | _lib.FLAG_CAPACITY)
    if np.any(bad):
        raise _lib.CapacityError(f"{int(np.count_nonzero(bad))} target(s) need the general path "
                                 f"(flags {np.unique(r.flags[bad != 0]).tolist()})")
    return r


def gather_results(local, group=None):
    """All-gather per-rank MultiTrackResults (targets in rank order)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    fields = {}
    for name in ("estimates", "ess", "occupied", "likelihood_evals"):
        a = np.ascontiguousarray(getattr(local, name))
        t = torch.from_numpy(a.astype(np.float64))
        n = torch.tensor([t.shape[0]])
        sizes = [torch.zeros_like(n) for _ in range(world)]
        dist.all_gather(sizes, n, group=group)
        mx = int(max(s.item() for s in sizes))
        pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=torch.float64)
        pad[:t.shape[0]] = t
        outs = [torch.zeros_like(pad) for _ in range(world)]
        dist.all_gather(outs, pad, group=group)
        fields[name] = np.concatenate([o[:int(s.item())].numpy() for o, s in zip(outs, sizes)])
    return fields


def multi_target_scene(n_targets, n_frames, width, seed=0, sigma=1.5, bg=10.0, margin=8):
    """Config-4 synthetic scene: spots at uniform positions, velocities
    N(0, 1) px/frame per axis, I0 ~ U[10, 40], one shared frame per time step
    with Poisson noise. Trajectories leaving the interior are redrawn
    (synthesis.py:108-121 convention). Returns (frames (K,W,W) float32,
    truth (T,K+1,5): state at k = 0..K, centres = truth[:, 0])."""
    rng = np.random.default_rng(seed)
    truth = np.empty((n_targets, n_frames + 1, 5))
    lo, hi = margin, width - 1 - margin
    for t in range(n_targets):
        while True:
            x0, y0 = rng.uniform(lo, hi, 2)
            vx, vy = rng.normal(0.0, 1.0, 2)
            i0 = rng.uniform(10.0, 40.0)
            ks = np.arange(n_frames + 1)
            xs, ys = x0 + vx * ks, y0 + vy * ks
            if xs.min() >= lo and xs.max() <= hi and ys.min() >= lo and ys.max() <= hi:
                truth[t, :, 0], truth[t, :, 1] = xs, ys
                truth[t, :, 2], truth[t, :, 3], truth[t, :, 4] = vx, vy, i0
                break
    frames = np.empty((n_frames, width, width), dtype=np.float32)
    r = int(np.ceil(5 * sigma))
    for k in range(n_frames):
        ideal = np.full((width, width), bg)
        for t in range(n_targets):
            x, y, i0 = truth[t, k + 1, 0], truth[t, k + 1, 1], truth[t, k + 1, 4]
            cx, cy = int(round(x)), int(round(y))
            xa, xb = max(cx - r, 0), min(cx + r + 1, width)
            ya, yb = max(cy - r, 0), min(cy + r + 1, width)
            gx = np.exp(-((np.arange(xa, xb) - x) ** 2) / (2 * sigma ** 2))
            gy = np.exp(-((np.arange(ya, yb) - y) ** 2) / (2 * sigma ** 2))
            ideal[ya:yb, xa:xb] += i0 * np.outer(gy, gx)
        frames[k] = rng.poisson(ideal)
    return frames, truth
