"""ctypes binding of libpcsir_b200.so (the C ABI in include/pcsir_b200.h).

This is the only module that talks to native code. There is no fallback: if
the shared library is missing or no CUDA device is visible, every call into
the filter step raises. Device buffers are torch CUDA tensors (plumbing only);
all arithmetic on the hot path runs in the sm_100a kernels of the library.
"""

import ctypes
import os
import pathlib
import threading

import torch

LIB_PATH = pathlib.Path(__file__).resolve().parent / "libpcsir_b200.so"

PCS_OK = 0
PCS_E_INVALID = 1
PCS_E_CUDA = 2
PCS_E_NOMEM = 3
PCS_E_CAPACITY = 4
E_CAPACITY = PCS_E_CAPACITY

FLAG_DEGENERATE = 1
FLAG_NONFINITE = 2
FLAG_CAPACITY = 4
FLAG_RANGE = 8

c_double = ctypes.c_double
c_int32 = ctypes.c_int32
c_int64 = ctypes.c_int64
c_uint32 = ctypes.c_uint32
c_uint64 = ctypes.c_uint64
c_void_p = ctypes.c_void_p
c_char_p = ctypes.c_char_p
P = ctypes.POINTER


class PcsGrid(ctypes.Structure):
    _fields_ = [("origin_x", c_double), ("origin_y", c_double),
                ("cell_width", c_double), ("cell_height", c_double),
                ("n_cols", c_int64), ("n_rows", c_int64)]


class PcsDynamics(ctypes.Structure):
    _fields_ = [("sigma_pos", c_double), ("sigma_vel", c_double),
                ("sigma_int", c_double), ("dt", c_double)]


class PcsSpot(ctypes.Structure):
    _fields_ = [("sigma_psf", c_double), ("i_bg", c_double), ("sigma_xi", c_double),
                ("halfwidth", c_int32), ("model", c_int32)]


class PcsInit(ctypes.Structure):
    _fields_ = [("center", c_double * 5), ("mode", c_int32), ("pad_", c_int32),
                ("width", c_double), ("sigma", c_double)]


class PcsTrackCfg(ctypes.Structure):
    _fields_ = [("method", c_int32), ("placement", c_int32), ("n_particles", c_int64),
                ("init", PcsInit), ("dyn", PcsDynamics), ("spot", PcsSpot),
                ("grid", PcsGrid), ("seed", c_uint64), ("frame0", c_uint32),
                ("use_graph", c_int32), ("threshold_fraction", c_double),
                ("scheme", c_int32), ("weighted_com", c_int32)]


class PcsTrackResult(ctypes.Structure):
    _fields_ = [("flags", c_uint32), ("first_bad_frame", c_int32),
                ("likelihood_evals", c_int64)]


# (name, restype, argtypes) — mirrors include/pcsir_b200.h exactly
_SIGNATURES = [
    ("pcs_last_error", c_char_p, []),
    ("pcs_version", c_int32, []),
    ("pcs_abi_struct_sizes", c_int32, [P(c_int64), c_int32]),
    ("pcs_device_info", c_int32, [c_int32, P(c_int32), P(c_int64), P(c_int32), P(c_int32)]),
    ("pcs_ctx_create", c_int32, [P(c_void_p), c_int32]),
    ("pcs_ctx_destroy", c_int32, [c_void_p]),
    ("pcs_philox_normals", c_int32, [c_uint64, c_uint32, c_int64, c_int64, c_void_p, c_int64, c_void_p]),
    ("pcs_philox_init_normals", c_int32, [c_uint64, c_int64, c_int64, c_void_p, c_int64, c_void_p]),
    ("pcs_philox_init_uniforms", c_int32, [c_uint64, c_int64, c_int64, c_void_p, c_int64, c_void_p]),
    ("pcs_philox_resample_u", c_double, [c_uint64, c_uint32]),
    ("pcs_philox_multinomial_points", c_int32, [c_uint64, c_uint32, c_int64, c_void_p, c_void_p]),
    ("pcs_render_frames", c_int32, [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int64,
                                    c_double, c_double, c_double, c_int32, c_double, c_uint64,
                                    c_uint32, c_void_p, c_void_p]),
    ("pcs_init_particles", c_int32, [P(PcsInit), c_uint64, c_int64, c_int64, c_void_p, c_int64, c_void_p]),
    ("pcs_propagate", c_int32, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, P(PcsDynamics),
                                c_uint64, c_uint32, c_int64, c_void_p]),
    ("pcs_propagate_given", c_int32, [c_void_p, c_void_p, c_int64, c_int64, c_void_p,
                                      P(PcsDynamics), c_void_p, c_int64, c_void_p]),
    ("pcs_gather", c_int32, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p]),
    ("pcs_spot_window_ssd_f64", c_int32, [c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p,
                                          c_int64, c_double, c_double, c_int32, c_void_p, c_void_p]),
    ("pcs_loglik", c_int32, [c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_int64,
                             P(PcsSpot), c_void_p, c_void_p]),
    ("pcs_partition", c_int32, [c_void_p, c_void_p, c_int64, c_int64, P(PcsGrid), c_void_p, c_void_p,
                                c_void_p, c_void_p, c_void_p, c_void_p, P(c_int64), c_void_p]),
    ("pcs_dummies", c_int32, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p,
                              c_void_p, c_int64, P(PcsGrid), c_int32, c_void_p, c_void_p, c_int64,
                              c_void_p]),
    ("pcs_weight_update", c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p,
                                    c_void_p]),
    ("pcs_normalize", c_int32, [c_void_p, c_void_p, c_int64, c_void_p, P(c_double), P(c_double),
                                P(c_int32), c_void_p]),
    ("pcs_estimate_ess", c_int32, [c_void_p, c_void_p, c_int64, c_void_p, c_int64, P(c_double),
                                   P(c_double), c_void_p]),
    ("pcs_resample_systematic", c_int32, [c_void_p, c_void_p, c_int64, c_double, c_void_p, c_void_p]),
    ("pcs_resample_multinomial", c_int32, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    ("pcs_cdf", c_int32, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    ("pcs_track", c_int32, [c_void_p, P(PcsTrackCfg), c_void_p, c_int64, c_int64, c_int64, c_void_p,
                            c_void_p, c_void_p, c_void_p, P(PcsTrackResult), c_void_p]),
    ("pcs_track_begin", c_int32, [c_void_p, P(PcsTrackCfg), c_int64, c_int64, c_void_p]),
    ("pcs_track_steps", c_int32, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p,
                                  c_void_p, c_void_p]),
    ("pcs_track_end", c_int32, [c_void_p, P(PcsTrackResult), c_void_p]),
    ("pcs_track_steps_timed", c_int32, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p,
                                        c_void_p, c_void_p, c_void_p, c_int32, c_void_p]),
    ("pcs_track_kernel_name", c_char_p, [c_void_p, c_int32]),
    ("pcs_track_launches_per_step", c_int32, [c_void_p]),
    ("pcs_track_debug", c_int32, [c_void_p, c_void_p, c_void_p]),
    ("pcs_track_info", c_int32, [c_void_p, c_void_p, c_int32, c_void_p]),
    ("pcs_bounds_deriv_max", c_int32, [c_int32, c_void_p, c_double, c_double, c_int64, c_double,
                                       c_double, c_int64, c_void_p, c_void_p]),
    ("pcs_bounds_midpoint", c_int32, [c_int32, c_void_p, c_void_p, c_int64, c_void_p, c_int64,
                                      c_void_p, c_void_p, c_int32, c_void_p, c_void_p]),
    ("pcs_make_dummy", c_int32, [c_void_p, c_int64, c_void_p, c_int32, c_void_p, c_void_p,
                                 c_void_p]),
    ("pcs_track_states", c_int32, [c_void_p, P(c_void_p), P(c_int64)]),
    ("pcs_mt_begin", c_int32, [c_void_p, P(PcsTrackCfg), c_int64, c_void_p, c_int64, c_int64,
                               c_int64, c_int64, c_void_p]),
    ("pcs_mt_step", c_int32, [c_void_p, c_void_p, c_int64, c_void_p]),
    ("pcs_mt_results", c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                 c_void_p, c_void_p]),
    ("pcs_shard_begin", c_int32, [c_void_p, P(PcsTrackCfg), c_int64, c_int64, c_int32, c_int32,
                                  c_int64, c_int64, c_int64, c_void_p]),
    ("pcs_shard_step1", c_int32, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p,
                                  c_void_p, c_void_p, c_void_p]),
    ("pcs_shard_export", c_int32, [c_void_p, c_void_p, c_void_p, c_void_p]),
    ("pcs_shard_import_bins", c_int32, [c_void_p, c_void_p, c_void_p, c_void_p]),
    ("pcs_shard_total", c_int32, [c_void_p, c_void_p, c_void_p]),
    ("pcs_shard_emit", c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("pcs_shard_unpack", c_int32, [c_void_p, c_void_p, c_void_p, c_void_p]),
    ("pcs_shard_prior", c_int32, [c_void_p, c_int32, c_void_p, c_void_p, c_void_p, c_void_p,
                                  c_void_p]),
    ("pcs_shard_route", c_int32, [c_void_p, c_void_p, c_void_p, c_void_p]),
    ("pcs_shard_serve", c_int32, [c_void_p, c_void_p, c_void_p, c_void_p]),
    ("pcs_shard_install", c_int32, [c_void_p, c_void_p, c_void_p]),
]

EXPORTED_SYMBOLS = [name for name, _, _ in _SIGNATURES]

_lib = None
_lock = threading.Lock()
_ctxs = {}


class NativeError(RuntimeError):
    """A C-ABI call failed (CUDA error, out of memory, bad argument)."""


class CapacityError(NativeError):
    """The fused path's bin window / occupied-bin capacity was exceeded."""


def load_library(path=None):
    """Load libpcsir_b200.so and bind every symbol; raises if anything is missing."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = pathlib.Path(path) if path else LIB_PATH
        if not p.exists():
            raise ImportError(
                f"{p} is missing: build the sm_100a extension first "
                "(python -c 'import __graft_entry__ as g; g.build()' or ./build.sh)")
        lib = ctypes.CDLL(str(p))
        for name, res, args in _SIGNATURES:
            fn = getattr(lib, name)  # AttributeError if the export is missing
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def lib():
    return _lib if _lib is not None else load_library()


def last_error():
    msg = lib().pcs_last_error()
    return msg.decode() if msg else ""


def check(rc, what="pcs call"):
    if rc == PCS_OK:
        return
    msg = last_error()
    if rc == PCS_E_INVALID:
        raise ValueError(f"{what}: {msg}")
    if rc == PCS_E_CAPACITY:
        raise CapacityError(f"{what}: capacity exceeded ({msg})")
    raise NativeError(f"{what} failed (status {rc}): {msg}")


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1310_5541_b200 needs a CUDA device (sm_100a); none is visible")


def device():
    require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def ctx():
    """Per-device pcs_ctx (scratch arena + fused-track state)."""
    dev = device()
    key = dev.index
    if key not in _ctxs:
        handle = c_void_p()
        check(lib().pcs_ctx_create(ctypes.byref(handle), key), "pcs_ctx_create")
        _ctxs[key] = handle
    return _ctxs[key]


def new_ctx():
    """A further pcs_ctx on the current device (its own scratch and track
    state), e.g. one per emulated rank of the sharded filter."""
    handle = c_void_p()
    check(lib().pcs_ctx_create(ctypes.byref(handle), device().index), "pcs_ctx_create")
    return handle


def stream():
    return c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    if t is None:
        return c_void_p(0)
    return c_void_p(t.data_ptr())


def device_info(index=0):
    sm = c_int32()
    l2 = c_int64()
    ma = c_int32()
    mi = c_int32()
    check(lib().pcs_device_info(index, ctypes.byref(sm), ctypes.byref(l2), ctypes.byref(ma),
                                ctypes.byref(mi)), "pcs_device_info")
    return {"sm_count": sm.value, "l2_bytes": l2.value, "cc": (ma.value, mi.value)}


LIK_F64 = 16   # pcs_spot_t.model flag: Poisson models in float64 (pcSIR cells)

TRACK_INFO_KEYS = ("s1_ctas", "s1_tile", "s1_tiles_per_warp", "rs_ctas", "rs_tiles_per_cta",
                   "sir_chunk", "s1_cell_flushes", "max_occupied", "cells_capacity",
                   "s1_cell_flush", "sir_ctas", "launches_per_frame")


def track_info():
    """pcs_track_info of the context's current / last fused track as a dict."""
    buf = (ctypes.c_int64 * 16)()
    check(lib().pcs_track_info(ctx(), buf, 16, stream()), "pcs_track_info")
    return {k: int(buf[i]) for i, k in enumerate(TRACK_INFO_KEYS)}


def loaded_library_path():
    return str(LIB_PATH) if _lib is not None else None


if os.environ.get("PCS_PRELOAD", "0") == "1":  # pragma: no cover
    load_library()
