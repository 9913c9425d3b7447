"""Gaussian-spot appearance model and the windowed residual likelihood.

Mirrors ``pcsir.imaging`` (imaging.py:1-146). Two evaluation forms:

* ``SpotLikelihood.batch(states, frame)`` — the reference's duck-typed
  operator: host (M,5) float64 states in, float64 likelihood values out,
  computed by the float64 device kernel ``pcs_spot_window_ssd_f64``
  (same operation order as _speedups.pyx:70-83).
* ``SpotLikelihood.loglik(soa, frame)`` — the float32 hot path used by the
  filter steps: device states in, device float32 log-likelihoods out.

``PoissonSpotLikelihood`` is the config-3 costly likelihood (new, not in the
reference): erf-integrated (or mid-point 4x4 supersampled) PSF with a Poisson
log-likelihood ratio against the background.
"""

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, kernels
from .state import I0, X, Y, StateVector


@dataclass(frozen=True)
class PsfParams:
    """Point-spread-function width and background level (imaging.py:19-30)."""

    sigma_psf: float
    i_bg: float = 0.0

    def __post_init__(self):
        if self.sigma_psf <= 0:
            raise ValueError("sigma_psf must be > 0")
        if self.i_bg < 0:
            raise ValueError("i_bg must be >= 0")


class ImageFrame:
    """One movie frame (imaging.py:33-55); ``pixels[y, x]``.

    Host pixels are kept as float64 like the reference; ``device()`` returns a
    cached float32 CUDA copy (exact for integer photon counts < 2^24).
    """

    def __init__(self, pixels, pixel_size_nm=67.0):
        if isinstance(pixels, torch.Tensor):
            self._dev = pixels.float().contiguous() if pixels.is_cuda else None
            pixels = pixels.detach().double().cpu().numpy()
        else:
            self._dev = None
        self.pixels = np.ascontiguousarray(pixels, dtype=np.float64)
        if self.pixels.ndim != 2:
            raise ValueError("pixels must be 2D")
        self.pixel_size_nm = pixel_size_nm

    @property
    def height(self):
        return self.pixels.shape[0]

    @property
    def width(self):
        return self.pixels.shape[1]

    def device(self):
        if self._dev is None:
            self._dev = torch.from_numpy(self.pixels.astype(np.float32)).to(_lib.device())
        return self._dev


def default_halfwidth(sigma_psf) -> int:
    """Window half-width covering three PSF standard deviations (imaging.py:58-60)."""
    return math.ceil(3.0 * sigma_psf)


@dataclass(frozen=True)
class LikelihoodParams:
    """Residual scale and window half-width (imaging.py:63-80)."""

    sigma_xi: float
    window_halfwidth: int

    def __post_init__(self):
        if self.sigma_xi <= 0:
            raise ValueError("sigma_xi must be > 0")
        if self.window_halfwidth < 0:
            raise ValueError("window_halfwidth must be >= 0")


def render_object(pos, i0, psf: PsfParams, at) -> float:
    """Ideal intensity of a spot at ``pos`` evaluated at ``at`` (imaging.py:83-92)."""
    dx, dy = at[0] - pos[0], at[1] - pos[1]
    return psf.i_bg + i0 * math.exp(-(dx * dx + dy * dy) / (2.0 * psf.sigma_psf ** 2))


def _clamped_span(coord, halfwidth, extent):
    """Inclusive [lo, hi] of the pixels within ``halfwidth`` of the pixel
    nearest to ``coord``, clamped into [0, extent - 1] (never empty)."""
    centre = int(np.floor(coord + 0.5))
    last = extent - 1
    return (min(max(centre - halfwidth, 0), last), min(max(centre + halfwidth, 0), last))


def window_bounds(frame: ImageFrame, x, y, halfwidth):
    """Clamped window (x_lo, x_hi, y_lo, y_hi), inclusive, never empty (imaging.py:95-103)."""
    return (*_clamped_span(x, halfwidth, frame.width), *_clamped_span(y, halfwidth, frame.height))


def window_pixel_count(frame: ImageFrame, x, y, halfwidth) -> int:
    x_lo, x_hi, y_lo, y_hi = window_bounds(frame, x, y, halfwidth)
    return (1 + x_hi - x_lo) * (1 + y_hi - y_lo)


class _DeviceLikelihood:
    """Shared device evaluation (float32 hot path) for the built-in models."""

    model = 0

    def spot_c(self, cells=False):
        """C description; ``cells``: the pcSIR per-cell form (the Poisson
        models in float64, PCS_LIK_F64 — few evaluations, |d log L| <= 1e-5)."""
        model = int(self.model) | (_lib.LIK_F64 if (cells and self.model != 0) else 0)
        return _lib.PcsSpot(float(self.psf.sigma_psf), float(self.psf.i_bg),
                            float(self.params.sigma_xi), int(self.params.window_halfwidth), model)

    def loglik(self, soa, frame: ImageFrame, count=True, cells=False):
        """Log-likelihood (float64) of each state column of ``soa`` (5,M) float32
        device; ``cells`` selects the pcSIR per-cell (dummy) form."""
        m = soa.shape[1]
        out = torch.empty(m, dtype=torch.float64, device=soa.device)
        if m:
            pix = frame.device()
            spot = self.spot_c(cells)
            soa = soa.contiguous()
            _lib.check(_lib.lib().pcs_loglik(
                _lib.ptr(pix), pix.shape[0], pix.shape[1], _lib.ptr(soa[X]), _lib.ptr(soa[Y]),
                _lib.ptr(soa[I0]), m, ctypes.byref(spot), _lib.ptr(out), _lib.stream()),
                "pcs_loglik")
        if count:
            self.evals += m
        return out


@dataclass
class SpotLikelihood(_DeviceLikelihood):
    """Windowed Gaussian-residual likelihood with an evaluation counter (imaging.py:111-140)."""

    psf: PsfParams
    params: LikelihoodParams
    evals: int = field(default=0, compare=False)
    model = 0

    def batch(self, states, frame: ImageFrame) -> np.ndarray:
        states = np.asarray(states, dtype=np.float64)
        ssd = kernels.spot_window_ssd(
            frame.pixels,
            np.ascontiguousarray(states[:, X]),
            np.ascontiguousarray(states[:, Y]),
            np.ascontiguousarray(states[:, I0]),
            self.psf.sigma_psf,
            self.psf.i_bg,
            self.params.window_halfwidth,
        )
        self.evals += states.shape[0]
        return np.exp(-ssd / (2.0 * self.params.sigma_xi ** 2))

    def __call__(self, state: StateVector, frame: ImageFrame) -> float:
        return float(self.batch(state.as_array()[None, :], frame)[0])


@dataclass
class PoissonSpotLikelihood(_DeviceLikelihood):
    """Config-3 likelihood (new): Poisson log-likelihood ratio vs background.

    lambda = bg + I0 * Ex(x) * Ey(y) over the clamped (2hw+1)^2 window;
    log L = sum_window [z log1p(mu/bg) - mu], mu = I0 Ex Ey (the full-frame
    Poisson log-likelihood up to a per-frame constant, lgamma term dropped).
    ``subpixel="erf"``: Ex is the exact pixel integral of the Gaussian
    (the 4x4 sub-pixel supersampled integral telescopes to it);
    ``subpixel="midpoint4"``: Ex is the 4-point mid-point average per axis.
    """

    psf: PsfParams
    params: LikelihoodParams
    subpixel: str = "erf"
    evals: int = field(default=0, compare=False)

    def __post_init__(self):
        if self.subpixel not in ("erf", "midpoint4"):
            raise ValueError("subpixel must be 'erf' or 'midpoint4'")
        if self.psf.i_bg <= 0:
            raise ValueError("the Poisson likelihood needs i_bg > 0")

    @property
    def model(self):
        return 1 if self.subpixel == "erf" else 2

    def batch(self, states, frame: ImageFrame) -> np.ndarray:
        st = np.asarray(states, dtype=np.float64)
        soa = torch.from_numpy(np.ascontiguousarray(st.T.astype(np.float32))).to(_lib.device())
        ll = self.loglik(soa, frame)
        return np.exp(ll.double().cpu().numpy())

    def __call__(self, state: StateVector, frame: ImageFrame) -> float:
        return float(self.batch(state.as_array()[None, :], frame)[0])


def likelihood(state: StateVector, frame: ImageFrame, psf: PsfParams,
               lp: LikelihoodParams) -> float:
    """One-shot evaluation of the windowed residual likelihood (imaging.py:143-146)."""
    return SpotLikelihood(psf, lp)(state, frame)
