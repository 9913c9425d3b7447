"""CPU oracle for the pcSIR / SIR filter step — TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and the CPU-baseline legs of
``bench.py`` may import this module, and only as the checker / the timed
CPU baseline. The product path (paper_1310_5541_b200) never imports it.

Two layers:

1. A numpy restatement of the reference algorithm (/root/reference/pkg/src/
   pcsir, each function cites the file:line it follows): float64 states,
   stable argsort + reduceat dummies, sequential cumsum + searchsorted
   resampling, a replayable RNG adapter. Pinned against golden vectors
   produced by the reference itself (tests/golden/make_golden.py) and against
   the reference tests' inline known answers.
2. The canonical exact conventions the device implements:
   exact-prefix cdf, exact per-bin sums, exact estimate / ESS / normaliser —
   restated in C (oracle/oracle.c, liboracle.so) so that bin counts, dummies
   and resampling indices can be compared bit-for-bit.

Parity protocol: each device stage is checked on the device's
own float32 inputs to that stage (upcast to float64) and the device's RNG
draws (replayed), because end-to-end trajectories diverge chaotically after
any rounding difference.
"""

import ctypes
import pathlib
import subprocess

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"

X, Y, VX, VY, I0 = range(5)

# --------------------------------------------------------------------------
# C library
# --------------------------------------------------------------------------
_lib = None


def build():
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = ctypes.CDLL(str(LIB))
        dp = ctypes.c_void_p
        i64 = ctypes.c_int64
        u64 = ctypes.c_uint64
        u32 = ctypes.c_uint32
        d = ctypes.c_double
        sig = {
            "orc_philox4x32": (None, [u64, dp, i64, dp]),
            "orc_propagate_normals": (None, [u64, u32, i64, i64, dp]),
            "orc_init_normals": (None, [u64, i64, i64, dp]),
            "orc_resample_u": (d, [u64, u32]),
            "orc_multinomial_points": (None, [u64, u32, i64, dp]),
            "orc_fixed_f32": (None, [dp, i64, ctypes.c_int, dp]),
            "orc_u128_to_double": (d, [u64, u64]),
            "orc_propagate": (None, [dp, dp, i64, d, d, d, d, dp]),
            "orc_propagate_f64": (None, [dp, dp, i64, d, d, d, d, dp]),
            "orc_spot_window_ssd": (None, [dp, i64, i64, dp, dp, dp, i64, d, d, i64, dp]),
            "orc_poisson_loglik": (None, [dp, i64, i64, dp, dp, dp, i64, d, d, i64, ctypes.c_int, dp]),
            "orc_cdf_exact": (None, [dp, i64, dp]),
            "orc_systematic_from_cdf": (None, [dp, i64, d, dp]),
            "orc_searchsorted_right": (None, [dp, i64, dp, i64, dp]),
            "orc_dummies_exact": (None, [dp, i64, dp, i64, dp, dp, dp]),
            "orc_normalize": (ctypes.c_int, [dp, i64, dp, dp, dp]),
            "orc_estimate_ess": (None, [dp, dp, i64, dp, dp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# --------------------------------------------------------------------------
# RNG: Philox restatement + replay adapter for the reference code
# --------------------------------------------------------------------------
def philox4x32(seed, counters):
    ctr = _c(counters, np.uint32).reshape(-1, 4)
    out = np.empty_like(ctr)
    lib().orc_philox4x32(seed, _p(ctr), ctr.shape[0], _p(out))
    return out


def propagate_normals(seed, frame, n, offset=0):
    """(5, n) float64 Box–Muller normals on the device's Philox uniforms."""
    out = np.empty((5, n))
    lib().orc_propagate_normals(seed, frame, offset, n, _p(out))
    return out


def init_normals(seed, n, offset=0):
    out = np.empty((2, n))
    lib().orc_init_normals(seed, offset, n, _p(out))
    return out


def resample_u(seed, frame):
    return lib().orc_resample_u(seed, frame)


def multinomial_points(seed, frame, n):
    out = np.empty(n)
    lib().orc_multinomial_points(seed, frame, n, _p(out))
    return out


class ReplayRng:
    """Duck-typed stand-in for numpy.random.Generator that returns recorded
    draws in call order. Supports exactly the calls the reference hot path
    makes: normal(loc, scale, size) (state.py:125,173), uniform(low, high,
    size) (state.py:171), random(size=None) (filtering.py:97,99)."""

    def __init__(self, normals=(), uniforms=(), randoms=()):
        self._normals = list(normals)
        self._uniforms = list(uniforms)
        self._randoms = list(randoms)

    def push_normal(self, z):
        self._normals.append(np.asarray(z, dtype=np.float64))

    def push_random(self, r):
        self._randoms.append(r)

    def normal(self, loc=0.0, scale=1.0, size=None):
        z = self._normals.pop(0)
        z = np.asarray(z, dtype=np.float64).reshape(size if size is not None else ())
        return loc + scale * z

    def uniform(self, low=0.0, high=1.0, size=None):
        u = np.asarray(self._uniforms.pop(0), dtype=np.float64).reshape(size)
        return low + (high - low) * u

    def random(self, size=None):
        r = self._randoms.pop(0)
        if size is None:
            return float(r)
        return np.asarray(r, dtype=np.float64).reshape(size)


class PhiloxReplay:
    """Generator stand-in that serves the device's counter-based draws in the
    reference's call order: the first ``normal(0, sigma, (n,2))`` is the init
    cloud (state.py:173), every ``normal(size=(N,5))`` is the next frame's
    propagation (state.py:125), ``random()`` / ``random(n)`` are the systematic
    offset / multinomial points of the frame just propagated
    (filtering.py:97,99). ``normals_fn(frame, n) -> (5, n)`` and
    ``init_fn(n) -> (2, n)`` may be overridden to replay the device's exact
    float32 normals (fetched through pcs_philox_normals)."""

    def __init__(self, seed, frame0=0, normals_fn=None, init_fn=None):
        self.seed = seed
        self.frame = frame0
        self.normals_fn = normals_fn or (lambda f, n: propagate_normals(seed, f, n))
        self.init_fn = init_fn or (lambda n: init_normals(seed, n))
        self._init_done = False

    def normal(self, loc=0.0, scale=1.0, size=None):
        n, width = size
        if width == 2 and not self._init_done:
            self._init_done = True
            z = np.asarray(self.init_fn(n), dtype=np.float64).T
        else:
            self._init_done = True
            z = np.asarray(self.normals_fn(self.frame, n), dtype=np.float64).T
            self.frame += 1
        return loc + scale * z

    def uniform(self, low=0.0, high=1.0, size=None):  # pragma: no cover - not on the configs
        raise NotImplementedError("uniform init is not replayed")

    def random(self, size=None):
        if size is None:
            return resample_u(self.seed, self.frame - 1)
        return multinomial_points(self.seed, self.frame - 1, int(size))


# --------------------------------------------------------------------------
# numpy restatement of the reference hot path (float64)
# --------------------------------------------------------------------------
def propagate_array(states, noise_scale, dt, normals_n5):
    """state.py:115-127 with the (N,5) standard normals given."""
    states = np.asarray(states, dtype=np.float64)
    out = states.copy()
    out[:, X] += states[:, VX] * dt
    out[:, Y] += states[:, VY] * dt
    out += np.asarray(normals_n5, dtype=np.float64) * np.asarray(noise_scale)
    np.maximum(out[:, I0], 0.0, out=out[:, I0])
    return out


def cell_indices(xs, ys, grid):
    """binning.py:61-67; grid = (ox, oy, lx, ly, ncols, nrows)."""
    ox, oy, lx, ly, ncols, nrows = grid
    ix = np.floor((np.asarray(xs, dtype=np.float64) - ox) / lx)
    iy = np.floor((np.asarray(ys, dtype=np.float64) - oy) / ly)
    ix = np.clip(ix, 0, ncols - 1).astype(np.int64)
    iy = np.clip(iy, 0, nrows - 1).astype(np.int64)
    return ix, iy


def partition(states, grid):
    """binning.py:97-112 -> (flat, order, unique, starts, counts)."""
    states = np.asarray(states, dtype=np.float64)
    ix, iy = cell_indices(states[:, X], states[:, Y], grid)
    flat = iy * grid[4] + ix
    order = np.argsort(flat, kind="stable")
    sorted_flat = flat[order]
    boundaries = np.flatnonzero(sorted_flat[1:] != sorted_flat[:-1]) + 1
    starts = np.concatenate(([0], boundaries))
    counts = np.diff(np.concatenate((starts, [len(flat)])))
    unique = sorted_flat[starts]
    return flat, order, unique, starts, counts


def bin_of_from_partition(n, order, counts):
    bin_of = np.empty(n, dtype=np.int32)
    bin_of[order] = np.repeat(np.arange(len(counts), dtype=np.int32), counts)
    return bin_of


def dummy_states(states, grid, order, unique, starts, counts, placement="com", weights=None):
    """binning.py:157-172 (reduceat CoM / weighted CoM / cell centre).

    ``weights`` is indexed exactly as the reference does (``weights[order]``,
    binning.py:160); note pc_sis_step passes ``pset.weights[order]``
    (binning.py:183), so a weighted-CoM step permutes the prior weights twice.
    The device path reproduces that behaviour."""
    states = np.asarray(states, dtype=np.float64)
    grouped = states[order]
    if weights is not None:
        w = np.asarray(weights, dtype=np.float64)[order]
        sums = np.add.reduceat(grouped * w[:, None], starts, axis=0)
        w_sums = np.add.reduceat(w, starts)
        dummies = sums / w_sums[:, None]
    else:
        dummies = np.add.reduceat(grouped, starts, axis=0) / counts[:, None]
    if placement == "coc":
        ox, oy, lx, ly, ncols, _ = grid
        ix, iy = unique % ncols, unique // ncols
        dummies[:, X] = ox + (ix + 0.5) * lx
        dummies[:, Y] = oy + (iy + 0.5) * ly
    return dummies


def spot_window_ssd_py(pixels, xs, ys, i0s, sigma_psf, i_bg, halfwidth):
    """kernels.py:24-40 (numpy fallback form), for small inputs."""
    height, width = pixels.shape
    n = xs.shape[0]
    out = np.empty(n)
    inv = 1.0 / (2.0 * sigma_psf * sigma_psf)
    for i in range(n):
        cx = int(np.floor(xs[i] + 0.5))
        cy = int(np.floor(ys[i] + 0.5))
        x_lo = min(max(cx - halfwidth, 0), width - 1)
        x_hi = min(max(cx + halfwidth, 0), width - 1)
        y_lo = min(max(cy - halfwidth, 0), height - 1)
        y_hi = min(max(cy + halfwidth, 0), height - 1)
        gx = np.exp(-((np.arange(x_lo, x_hi + 1) - xs[i]) ** 2) * inv)
        gy = np.exp(-((np.arange(y_lo, y_hi + 1) - ys[i]) ** 2) * inv)
        resid = pixels[y_lo:y_hi + 1, x_lo:x_hi + 1] - (i0s[i] * np.outer(gy, gx) + i_bg)
        out[i] = np.sum(resid * resid)
    return out


def spot_window_ssd(pixels, xs, ys, i0s, sigma_psf, i_bg, halfwidth):
    """_speedups.pyx:42-83 restated in C (same loop order), float64."""
    pixels = _c(pixels, np.float64)
    xs, ys, i0s = (_c(a, np.float64) for a in (xs, ys, i0s))
    out = np.empty(xs.shape[0])
    lib().orc_spot_window_ssd(_p(pixels), pixels.shape[0], pixels.shape[1], _p(xs), _p(ys),
                              _p(i0s), xs.shape[0], float(sigma_psf), float(i_bg),
                              int(halfwidth), _p(out))
    return out


def loglik_gauss(pixels, xs, ys, i0s, sigma_psf, i_bg, halfwidth, sigma_xi):
    """log of imaging.py:137: -ssd / (2 sigma_xi^2)."""
    return -spot_window_ssd(pixels, xs, ys, i0s, sigma_psf, i_bg, halfwidth) / (2.0 * sigma_xi ** 2)


def loglik_poisson(pixels, xs, ys, i0s, sigma_psf, i_bg, halfwidth, model=1):
    """R19 (config 3, new): Poisson log-likelihood ratio, brute-force 4x4 sub-pixels."""
    pixels = _c(pixels, np.float64)
    xs, ys, i0s = (_c(a, np.float64) for a in (xs, ys, i0s))
    out = np.empty(xs.shape[0])
    lib().orc_poisson_loglik(_p(pixels), pixels.shape[0], pixels.shape[1], _p(xs), _p(ys),
                             _p(i0s), xs.shape[0], float(sigma_psf), float(i_bg), int(halfwidth),
                             int(model), _p(out))
    return out


def render_ideal(spots, width, height, sigma_psf, i_bg):
    """Ideal frame of several spots (synthesis.py:124-130, render_clean_frame,
    summed over spots): i_bg + sum_s I0_s outer(gy_s, gx_s), float64 over the
    whole frame. ``spots``: (S, 3) (x, y, I0)."""
    out = np.full((height, width), float(i_bg))
    xs, ys = np.arange(width, dtype=np.float64), np.arange(height, dtype=np.float64)
    for x, y, i0 in np.asarray(spots, dtype=np.float64).reshape(-1, 3):
        gx = np.exp(-((xs - x) ** 2) / (2.0 * sigma_psf ** 2))
        gy = np.exp(-((ys - y) ** 2) / (2.0 * sigma_psf ** 2))
        out += i0 * np.outer(gy, gx)
    return out


def normalize(weights):
    """filtering.py:75-85."""
    w_max = weights.max()
    if not np.isfinite(w_max) or w_max <= 0:
        raise ZeroDivisionError("degenerate")
    scaled = weights / w_max
    return scaled / scaled.sum()


def effective_sample_size(weights):
    """filtering.py:88-90."""
    return 1.0 / float(np.sum(weights ** 2))


def resample_indices_reference(weights, n, scheme, rng):
    """filtering.py:93-100 verbatim semantics (sequential float64 cumsum)."""
    cdf = np.cumsum(weights)
    cdf[-1] = 1.0
    if scheme == "multinomial":
        points = rng.random(n)
    else:
        points = (rng.random() + np.arange(n)) / n
    return np.searchsorted(cdf, points, side="right")


# --------------------------------------------------------------------------
# canonical exact conventions (C) — what the device must equal bit-for-bit
# --------------------------------------------------------------------------
def cdf_exact(w32):
    w = _c(w32, np.float32)
    out = np.empty(w.shape[0])
    lib().orc_cdf_exact(_p(w), w.shape[0], _p(out))
    return out


def systematic_exact(w32, u):
    """Canonical systematic ancestors: exact-prefix cdf, cdf[-1]=1, points
    RN(RN(u+j)/n), searchsorted right, index n clamped to n-1."""
    cdf = cdf_exact(w32)
    anc = np.empty(cdf.shape[0], dtype=np.int32)
    lib().orc_systematic_from_cdf(_p(cdf), cdf.shape[0], float(u), _p(anc))
    return anc


def multinomial_exact(w32, points):
    cdf = cdf_exact(w32)
    pts = _c(points, np.float64)
    anc = np.empty(pts.shape[0], dtype=np.int32)
    lib().orc_searchsorted_right(_p(cdf), cdf.shape[0], _p(pts), pts.shape[0], _p(anc))
    return anc


def dummies_exact(soa32, bin_of, counts, prior_w=None):
    """Canonical per-bin dummies (5, M) float32 from exact integer sums."""
    s = _c(soa32, np.float32)
    n = s.shape[1]
    b = _c(bin_of, np.int32)
    cnt = _c(counts, np.int64)
    m = cnt.shape[0]
    out = np.empty((5, m), dtype=np.float32)
    pw = None if prior_w is None else _c(prior_w, np.float32)
    lib().orc_dummies_exact(_p(s), n, _p(b), m, _p(cnt), None if pw is None else _p(pw), _p(out))
    return out


def normalize_exact(logw):
    lw = _c(logw, np.float64)
    w = np.empty(lw.shape[0], dtype=np.float32)
    m = ctypes.c_double()
    s = ctypes.c_double()
    deg = lib().orc_normalize(_p(lw), lw.shape[0], _p(w), ctypes.byref(m), ctypes.byref(s))
    if deg:
        raise ZeroDivisionError("degenerate")
    return w, m.value, s.value


def estimate_ess_exact(soa32, w32):
    s = _c(soa32, np.float32)
    w = _c(w32, np.float32)
    est = np.empty(5)
    ess = ctypes.c_double()
    lib().orc_estimate_ess(_p(s), _p(w), w.shape[0], _p(est), ctypes.byref(ess))
    return est, ess.value


def propagate_f32(soa32, z32, sigma_pos, sigma_vel, sigma_int, dt):
    """state.py:115-127 in the device's canonical float32 form (one rounding
    per fused multiply-add, float32 parameters; oracle.c orc_propagate) —
    the bit-exact target of the device propagation."""
    s = _c(soa32, np.float32)
    z = _c(z32, np.float32)
    out = np.empty_like(s)
    lib().orc_propagate(_p(s), _p(z), s.shape[1], sigma_pos, sigma_vel, sigma_int, dt, _p(out))
    return out


def propagate_f64_order(soa32, z32, sigma_pos, sigma_vel, sigma_int, dt):
    """state.py:115-127 on the upcast float32 inputs in numpy's float64
    order, rounded once to float32 (the reference's values on these inputs)."""
    s = _c(soa32, np.float32)
    z = _c(z32, np.float32)
    out = np.empty_like(s)
    lib().orc_propagate_f64(_p(s), _p(z), s.shape[1], sigma_pos, sigma_vel, sigma_int, dt,
                            _p(out))
    return out


# --------------------------------------------------------------------------
# whole-filter restatement (filtering.py:148-182, binning.py:175-226) —
# used for the CPU baseline timing and the end-to-end oracle comparison
# --------------------------------------------------------------------------
class SpotModel:
    def __init__(self, sigma_psf, i_bg, sigma_xi, halfwidth, model="gauss", ssd=None):
        self.sigma_psf = sigma_psf
        self.i_bg = i_bg
        self.sigma_xi = sigma_xi
        self.halfwidth = halfwidth
        self.model = model
        self.evals = 0
        self._ssd = ssd or spot_window_ssd

    def batch(self, states, pixels):
        """imaging.py:125-137 (linear likelihood)."""
        self.evals += states.shape[0]
        if self.model == "gauss":
            ssd = self._ssd(pixels, np.ascontiguousarray(states[:, X]),
                            np.ascontiguousarray(states[:, Y]),
                            np.ascontiguousarray(states[:, I0]), self.sigma_psf, self.i_bg,
                            self.halfwidth)
            return np.exp(-ssd / (2.0 * self.sigma_xi ** 2))
        ll = loglik_poisson(pixels, states[:, X], states[:, Y], states[:, I0], self.sigma_psf,
                            self.i_bg, self.halfwidth, 1 if self.model == "erf" else 2)
        return np.exp(ll - ll.max())  # relative likelihood (constant cancels)


def track(frames, n, init_center, init_sigma, noise_scale, dt, lik, rng, grid=None,
          placement="com", threshold_fraction=1.0, scheme="systematic"):
    """filtering.py:148-173 with sis_step (grid None) or pc_sis_step
    (binning.py:175-195). ``rng`` is a numpy Generator or a ReplayRng."""
    states = np.tile(np.asarray(init_center, dtype=np.float64), (n, 1))
    if init_sigma > 0:
        states[:, (X, Y)] += rng.normal(0.0, init_sigma, size=(n, 2))
    weights = np.full(n, 1.0 / n)
    k_frames = len(frames)
    estimates = np.empty((k_frames, 5))
    ess_log = np.empty(k_frames)
    resampled = np.zeros(k_frames, dtype=bool)
    threshold = threshold_fraction * n
    for k, pixels in enumerate(frames):
        states = propagate_array(states, noise_scale, dt, rng.normal(size=states.shape))
        if grid is None:
            weights = weights * lik.batch(states, pixels)
        else:
            _, order, unique, starts, counts = partition(states, grid)
            dummies = dummy_states(states, grid, order, unique, starts, counts, placement)
            cell_lik = lik.batch(dummies, pixels)
            multiplier = np.empty(n)
            multiplier[order] = np.repeat(cell_lik, counts)
            weights = weights * multiplier
        weights = normalize(weights)
        estimates[k] = weights @ states
        ess_log[k] = effective_sample_size(weights)
        if ess_log[k] < threshold:
            idx = resample_indices_reference(weights, n, scheme, rng)
            states = states[idx]
            weights = np.full(n, 1.0 / n)
            resampled[k] = True
    return estimates, ess_log, resampled, lik.evals


# --------------------------------------------------------------------------
# reference compiled kernel (oracle/_ref, built from the reference .pyx)
# --------------------------------------------------------------------------
def reference_ssd_kernel():
    """The reference's own compiled Cython kernel if oracle/_ref holds it."""
    import importlib.util
    ref = HERE / "_ref"
    for so in sorted(ref.glob("_speedups*.so")) if ref.exists() else []:
        spec = importlib.util.spec_from_file_location("_speedups", so)
        mod = importlib.util.module_from_spec(spec)
        try:
            spec.loader.exec_module(mod)
        except ImportError:
            return None
        return mod.spot_window_ssd
    return None
