"""The reference's likelihood operator, served by the sm_100a kernel.

``spot_window_ssd`` keeps the signature and window convention of
``pcsir.kernels.spot_window_ssd`` (kernels.py:84-94, _speedups.pyx:17-85):
float64 (H,W) pixels and float64 state columns in, float64 SSDs out. The
computation runs in ``pcs_spot_window_ssd_f64`` on the GPU; there is no
backend registry and no host fallback (the reference's ``python`` /
``compiled`` switch has no counterpart here). ``available_backends`` /
``active_backend`` / ``set_backend`` exist only so callers of the reference
API keep importing; the single backend is ``"cuda"``.
"""

import numpy as np
import torch

from . import _lib

BACKEND = "cuda"
COMPILED_AVAILABLE = True


def available_backends():
    return [BACKEND]


def active_backend():
    return BACKEND


def set_backend(name):
    if name in (None, "auto", BACKEND):
        return BACKEND
    raise ValueError(f"unknown kernel backend {name!r} (have: {[BACKEND]})")


def spot_window_ssd(pixels, xs, ys, i0s, sigma_psf, i_bg, halfwidth, backend=None):
    """Batched windowed SSD between a frame and predicted Gaussian spots (kernels.py:84-94)."""
    if backend not in (None, BACKEND, "auto"):
        raise ValueError(f"unknown kernel backend {backend!r}")
    pixels = np.ascontiguousarray(pixels, dtype=np.float64)
    if pixels.ndim != 2:
        raise ValueError("pixels must be 2D")
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    ys = np.ascontiguousarray(ys, dtype=np.float64)
    i0s = np.ascontiguousarray(i0s, dtype=np.float64)
    n = xs.shape[0]
    if ys.shape != (n,) or i0s.shape != (n,):
        raise ValueError("xs, ys and i0s must have the same length")
    dev = _lib.device()
    out = torch.empty(n, dtype=torch.float64, device=dev)
    if n:
        pix = torch.from_numpy(pixels).to(dev)
        tx = torch.from_numpy(xs).to(dev)
        ty = torch.from_numpy(ys).to(dev)
        ti = torch.from_numpy(i0s).to(dev)
        _lib.check(_lib.lib().pcs_spot_window_ssd_f64(
            _lib.ptr(pix), pixels.shape[0], pixels.shape[1], _lib.ptr(tx), _lib.ptr(ty),
            _lib.ptr(ti), n, float(sigma_psf), float(i_bg), int(halfwidth), _lib.ptr(out),
            _lib.stream()), "pcs_spot_window_ssd_f64")
    return out.cpu().numpy()
