"""GPU scene synthesis for the benchmark scenes.

Device counterpart of the reference's frame rendering
(pkg/src/pcsir/synthesis.py:124-150): ``render_clean_frame`` (ideal
Gaussian-spot frame on a constant background) and ``render_sequence``
(Poisson measurement noise per pixel, optional Gaussian read noise clamped
at 0), generalised to several spots per frame (config 4). Frames are
rendered by ``pcs_render_frames`` straight into device memory, so the
4096x4096 (c5) and 2048x2048 x 4096-spot (c4) scenes cost milliseconds
instead of host ``rng.poisson`` minutes, and no host->device copy.

The ideal frame sums each spot's I0 gx gy over a +-ceil(window_sigmas * sigma)
window as an exact fixed-point (2^-32) sum, i.e. independent of spot order;
it matches the reference's float64 ``render_clean_frame`` to ~1e-9
(tests/test_gpu_synthesis.py against tests/golden/synth.npz). The noise
stream is Philox (seed, pixel, frame): the reference's numpy
``Generator.poisson`` stream cannot be reproduced, only its law (checked
statistically).
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .imaging import ImageFrame, PsfParams

WINDOW_SIGMAS = 8.0   # exp(-32) ~ 1e-14: far below the 2^-32 accumulation step


@dataclass(frozen=True)
class SceneConfig:
    """Rendering part of the reference's SceneConfig (synthesis.py:31-62)."""

    psf: PsfParams
    frames: int = 50
    width: int = 512
    height: int = 512
    read_noise_std: float = 0.0
    noise: bool = True
    seed: int = 0

    def __post_init__(self):
        if self.frames < 1:
            raise ValueError("frames must be >= 1")
        if self.width < 1 or self.height < 1:
            raise ValueError("frame size must be positive")
        if self.read_noise_std < 0:
            raise ValueError("read_noise_std must be >= 0")


def render_frames(spots, width, height, psf, noise=True, seed=0, frame0=0,
                  read_noise_std=0.0, window_sigmas=WINDOW_SIGMAS):
    """Render K frames on the device.

    ``spots``: (K, S, >=3) or (K, >=3) array-like of (x, y, I0[, ...]) per
    spot and frame (states with I0 in column 4 are accepted as (K, S, 5)).
    Returns a float32 CUDA tensor (K, height, width)."""
    a = np.asarray(spots, dtype=np.float64)
    if a.ndim == 2:
        a = a[:, None, :]
    if a.ndim != 3 or a.shape[2] < 3:
        raise ValueError("spots must be (K, S, 3) or (K, 3) (x, y, I0)")
    xyz = a[:, :, [0, 1, 4]] if a.shape[2] >= 5 else a[:, :, :3]
    k, s = xyz.shape[0], xyz.shape[1]
    dev = torch.from_numpy(np.ascontiguousarray(xyz)).cuda()
    out = torch.empty((k, height, width), dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib().pcs_render_frames(
        _lib.ctx(), _lib.ptr(dev), s, k, width, height, float(psf.sigma_psf), float(psf.i_bg),
        float(window_sigmas), 1 if noise else 0, float(read_noise_std), int(seed) & (2 ** 64 - 1),
        int(frame0) & 0xFFFFFFFF, _lib.ptr(out), _lib.stream()), "pcs_render_frames")
    return out


def render_clean_frame(state, cfg: SceneConfig) -> torch.Tensor:
    """Ideal (noise-free) frame for one truth state (synthesis.py:124-130)."""
    return render_frames(np.asarray(state, dtype=np.float64)[None, :], cfg.width, cfg.height,
                         cfg.psf, noise=False)[0]


def render_sequence(truth_states, cfg: SceneConfig, seed=None) -> list:
    """Noisy frames for a trajectory (synthesis.py:133-150): one ImageFrame
    per state row, Poisson per pixel (+ optional read noise), device-backed."""
    states = np.atleast_2d(np.asarray(truth_states, dtype=np.float64))
    frames = render_frames(states, cfg.width, cfg.height, cfg.psf, noise=cfg.noise,
                           seed=cfg.seed if seed is None else seed,
                           read_noise_std=cfg.read_noise_std)
    return [ImageFrame(frames[k]) for k in range(frames.shape[0])]


def spot_scene(n_frames, width, start, i0=20.0, velocity=(0.5, 0.0), psf=PsfParams(1.5, 10.0),
               seed=0, noise=True):
    """Benchmark scene of configs 1-3 and 5: one spot moving at constant
    velocity; returns (frames (K, W, W) float32 CUDA tensor, truth (K, 2))."""
    x0, y0 = start
    ks = np.arange(1, n_frames + 1)
    truth = np.stack([x0 + velocity[0] * ks, y0 + velocity[1] * ks], axis=1)
    spots = np.stack([truth[:, 0], truth[:, 1], np.full(n_frames, float(i0))], axis=1)
    return render_frames(spots, width, width, psf, noise=noise, seed=seed), truth


def multi_target_truth(n_targets, n_frames, width, seed=0, margin=8):
    """Config-4 trajectories (same law as multitarget.multi_target_scene):
    uniform interior start, velocity N(0, 1) px/frame per axis, I0 ~ U[10, 40],
    straight lines redrawn until they stay inside; (T, K+1, 5)."""
    rng = np.random.default_rng(seed)
    truth = np.empty((n_targets, n_frames + 1, 5))
    lo, hi = margin, width - 1 - margin
    ks = np.arange(n_frames + 1)
    for t in range(n_targets):
        while True:
            x0, y0 = rng.uniform(lo, hi, 2)
            vx, vy = rng.normal(0.0, 1.0, 2)
            i0 = rng.uniform(10.0, 40.0)
            xs, ys = x0 + vx * ks, y0 + vy * ks
            if xs.min() >= lo and xs.max() <= hi and ys.min() >= lo and ys.max() <= hi:
                truth[t, :, 0], truth[t, :, 1] = xs, ys
                truth[t, :, 2], truth[t, :, 3], truth[t, :, 4] = vx, vy, i0
                break
    return truth


def multi_target_scene_device(n_targets, n_frames, width, seed=0, psf=PsfParams(1.5, 10.0)):
    """Config-4 scene rendered on the device: frames (K, W, W) float32 CUDA
    tensor and truth (T, K+1, 5) (state at k = 0..K; frame k shows k+1)."""
    truth = multi_target_truth(n_targets, n_frames, width, seed)
    spots = np.ascontiguousarray(truth[:, 1:, :].transpose(1, 0, 2))   # (K, T, 5)
    return render_frames(spots, width, width, psf, noise=True, seed=seed), truth
