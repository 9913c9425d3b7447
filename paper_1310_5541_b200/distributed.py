"""Particle-sharded giant filter (BASELINE config 5; new — the reference is
single-process).

One filter of N particles is split across the ranks of a torch.distributed
group (one process per GPU, NCCL over NVLink): rank r owns the contiguous
global index range [r*n, (r+1)*n). Per frame the ranks exchange exactly what
the algorithm needs and nothing else:

  1. all-reduce MIN/MAX of the local occupied-cell bounding boxes (4 ints);
  2. all-reduce SUM of the per-cell accumulators over that window, carried as
     int64 limbs of the exact int128 sums — integer addition is associative,
     so the dummies are bit-identical for every rank count;
  3. every rank runs the same bins stage (dummies, likelihood per occupied
     cell, normaliser, estimate, ESS, resampling decision) on the same sums;
  4. all-gather of the ranks' exact cumulative-weight totals (u128) gives each
     rank its global cdf offset (distributed systematic resampling);
  5. all-to-all of the resampled states whose output slot belongs to another
     rank (monotone ancestors: one contiguous chunk per rank pair).

Philox counters use the global particle index, so the random draws — and
therefore every result — are the same for any number of ranks as for one GPU.

The per-rank compute is behind ``ShardOps``: ``DeviceShardOps`` (the product:
C-ABI kernels on the rank's GPU) or a CPU stand-in used by the gloo tests.
"""

import ctypes
import math

import numpy as np
import torch
import torch.distributed as dist

from . import _lib

FX_CDF = 120
LIMBS = 16


# ---------------------------------------------------------------------------
# exact host-side restatement of the device slot search (first_slot_at_or_above)
# ---------------------------------------------------------------------------
def cdf_value(prefix_int):
    """CANONICAL c = RN64(prefix) * 2^-120 (Python int -> float is correctly rounded)."""
    return math.ldexp(float(prefix_int), -FX_CDF)


def first_slot(c, u, n):
    """Smallest j in [0, n] with RN(RN(u + j) / n) >= c (slot n := +inf)."""
    nd = float(n)
    g = math.ceil(c * nd - u)
    j = 0 if not g > 0 else (n if g >= nd else int(g))
    while j > 0 and (u + float(j - 1)) / nd >= c:
        j -= 1
    while j < n and (u + float(j)) / nd < c:
        j += 1
    return j


def slot_ranges(totals, u, n_global, do_resample):
    """Global output-slot range [lo, hi) emitted by each rank's particles."""
    p = len(totals)
    n_local = n_global // p
    if not do_resample:
        return [(r * n_local, (r + 1) * n_local) for r in range(p)], [0] * p
    prefix = [0] * (p + 1)
    for r in range(p):
        prefix[r + 1] = prefix[r] + totals[r]
    lo = [0] + [first_slot(cdf_value(prefix[r]), u, n_global) for r in range(1, p)]
    hi = lo[1:] + [n_global]
    return list(zip(lo, hi)), prefix[:p]


def exchange_plan(ranges, n_global, p):
    """send[r][q] = (first index into rank r's emitted slots, count) going to rank q."""
    n_local = n_global // p
    plan = []
    for r in range(p):
        lo, hi = ranges[r]
        row = []
        for q in range(p):
            a, b = max(lo, q * n_local), min(hi, (q + 1) * n_local)
            row.append((a - lo, max(0, b - a)))
        plan.append(row)
    return plan


class ShardOps:
    """One rank's compute for the sharded step (see DeviceShardOps)."""

    def begin(self, cfg, height, width, idx_off, n_global, slot_cap, seed):
        raise NotImplementedError

    def step1(self, frame, k):
        """propagate + exact local cell sums; -> (bbox[4] ix0, ix1, iy0, iy1, n_occupied)"""
        raise NotImplementedError

    def export(self, window):
        raise NotImplementedError

    def import_bins(self, window, limbs):
        raise NotImplementedError

    def scan(self):
        """-> (exact local cumulative-weight total as int, do_resample)"""
        raise NotImplementedError

    def emit(self, prefix, slot_lo):
        raise NotImplementedError

    def gather(self, first, count):
        raise NotImplementedError

    def set_states(self, soa):
        raise NotImplementedError

    def advance(self):
        raise NotImplementedError

    def outputs(self):
        """-> (estimates (K,5), ess (K,), resampled (K,), occupied (K,)) host arrays"""
        raise NotImplementedError


class DeviceShardOps(ShardOps):
    """Product implementation: the rank's GPU through the C ABI (pcs_shard_*)."""

    def __init__(self, n_frames):
        self.n_frames = n_frames

    def begin(self, cfg, height, width, idx_off, n_global, slot_cap, seed):
        self.dev = _lib.device()
        self.n_local = cfg.n_particles
        self.est = torch.empty((self.n_frames, 5), dtype=torch.float64, device=self.dev)
        self.ess = torch.empty(self.n_frames, dtype=torch.float64, device=self.dev)
        self.res = torch.empty(self.n_frames, dtype=torch.uint8, device=self.dev)
        self.occ = torch.empty(self.n_frames, dtype=torch.int64, device=self.dev)
        c = _lib.PcsTrackCfg()
        c.method = 1
        c.placement = 1 if cfg.placement.value == "coc" else 0
        c.n_particles = cfg.n_particles
        c.init = cfg.init.to_c()
        c.dyn = cfg.dynamics.to_c()
        c.spot = cfg.likelihood.spot_c(cells=True)
        c.grid = cfg.grid.to_c()
        c.seed = seed
        c.frame0 = 0
        c.use_graph = 0
        self.cfg_c = c
        _lib.check(_lib.lib().pcs_shard_begin(_lib.ctx(), ctypes.byref(c), height, width, idx_off,
                                              n_global, slot_cap, _lib.stream()),
                   "pcs_shard_begin")

    def step1(self, frame, k):
        box = (ctypes.c_int64 * 5)()
        _lib.check(_lib.lib().pcs_shard_step1(
            _lib.ctx(), _lib.ptr(frame), k, _lib.ptr(self.est[k:]), _lib.ptr(self.ess[k:]),
            _lib.ptr(self.res[k:]), _lib.ptr(self.occ[k:]), box, _lib.stream()), "pcs_shard_step1")
        if box[4] > 16384:
            raise _lib.CapacityError("more occupied cells than the fused bins stage holds")
        return list(box[:4]), int(box[4])

    def export(self, window):
        x0, y0, nx, ny = window
        limbs = torch.empty((nx * ny, LIMBS), dtype=torch.int64, device=self.dev)
        _lib.check(_lib.lib().pcs_shard_export(_lib.ctx(), x0, y0, nx, ny, _lib.ptr(limbs),
                                               _lib.stream()), "pcs_shard_export")
        return limbs

    def import_bins(self, window, limbs):
        x0, y0, nx, ny = window
        _lib.check(_lib.lib().pcs_shard_import_bins(_lib.ctx(), x0, y0, nx, ny, _lib.ptr(limbs),
                                                    _lib.stream()), "pcs_shard_import_bins")

    def scan(self):
        lo, hi, dr = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_int32()
        _lib.check(_lib.lib().pcs_shard_scan(_lib.ctx(), ctypes.byref(lo), ctypes.byref(hi),
                                             ctypes.byref(dr), _lib.stream()), "pcs_shard_scan")
        return (hi.value << 64) | lo.value, bool(dr.value)

    def emit(self, prefix, slot_lo):
        anc = ctypes.c_void_p()
        _lib.check(_lib.lib().pcs_shard_emit(_lib.ctx(), prefix & (2 ** 64 - 1), prefix >> 64,
                                             slot_lo, ctypes.byref(anc), _lib.stream()),
                   "pcs_shard_emit")

    def gather(self, first, count):
        out = torch.empty((5, count), dtype=torch.float32, device=self.dev)
        _lib.check(_lib.lib().pcs_shard_gather(_lib.ctx(), first, count, _lib.ptr(out),
                                               _lib.stream()), "pcs_shard_gather")
        return out

    def set_states(self, soa):
        soa = soa.contiguous()
        _lib.check(_lib.lib().pcs_shard_set_states(_lib.ctx(), _lib.ptr(soa), _lib.stream()),
                   "pcs_shard_set_states")

    def advance(self):
        _lib.check(_lib.lib().pcs_shard_advance(_lib.ctx(), _lib.stream()), "pcs_shard_advance")

    def outputs(self):
        torch.cuda.synchronize()
        return (self.est.cpu().numpy(), self.ess.cpu().numpy(),
                self.res.cpu().numpy().astype(bool), self.occ.cpu().numpy())

    def resample_u(self, seed, frame):
        return float(_lib.lib().pcs_philox_resample_u(seed, frame & 0xFFFFFFFF))


def max_over_ranks(value, group=None):
    """The largest of every rank's ``value`` (a float), e.g. a device-timed
    duration, so that a multi-GPU throughput is the whole job's units over
    the slowest rank's time. A one-element all-reduce MAX on the backend's
    device (CUDA tensor for nccl, CPU tensor for gloo); identity when
    torch.distributed is not initialised."""
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    dev = torch.device("cuda", torch.cuda.current_device()) \
        if dist.get_backend(group) == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def _all_reduce_box(box, group, device):
    t = torch.tensor([-box[0], box[1], -box[2], box[3]], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    v = t.tolist()
    return -v[0], v[1], -v[2], v[3]


def sharded_pcsir_track(frames, cfg, seed, ops, group=None, slot_slack=2.0, comm_device=None):
    """Run pcSIR over the ranks of ``group``; every rank returns the same
    TrackResult-like tuple (estimates, ess, resampled, likelihood_evals).

    ``frames``: (K,H,W) float32 tensor on the rank's device (the frames are
    replicated: every rank evaluates the same occupied cells). ``cfg`` is a
    PcFilterConfig with the GLOBAL n_particles (divisible by the world size).
    """
    r_cfg = cfg.resampling
    if r_cfg.threshold_fraction != 1.0 or r_cfg.scheme != "systematic":
        raise ValueError("the sharded filter resamples every frame (systematic, "
                         "threshold_fraction=1.0); use pcsir_track on one GPU otherwise")
    p = dist.get_world_size(group)
    r = dist.get_rank(group)
    n_global = cfg.n_particles
    if n_global % p:
        raise ValueError("n_particles must be divisible by the number of ranks")
    n_local = n_global // p
    from dataclasses import replace
    local_cfg = replace(cfg, n_particles=n_local)
    k_frames, h, w = frames.shape
    slot_cap = int(n_local * slot_slack) + 64
    ops.begin(local_cfg, h, w, r * n_local, n_global, slot_cap, seed)
    dev = comm_device if comm_device is not None else (
        torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl"
        else torch.device("cpu"))
    for k in range(k_frames):
        box, _ = ops.step1(frames[k], k)
        ix0, ix1, iy0, iy1 = _all_reduce_box(box, group, dev)
        window = (ix0, iy0, ix1 - ix0 + 1, iy1 - iy0 + 1)
        limbs = ops.export(window)
        lt = limbs.to(dev)
        dist.all_reduce(lt, op=dist.ReduceOp.SUM, group=group)
        ops.import_bins(window, lt.to(limbs.device))
        total, do_res = ops.scan()
        if not do_res:
            ops.advance()
            continue
        tt = torch.tensor([total & (2 ** 62 - 1), total >> 62], dtype=torch.int64, device=dev)
        gathered = [torch.zeros_like(tt) for _ in range(p)]
        dist.all_gather(gathered, tt, group=group)
        totals = [int(g[0].item()) + (int(g[1].item()) << 62) for g in gathered]
        u = ops.resample_u(seed, k)
        ranges, prefixes = slot_ranges(totals, u, n_global, True)
        if ranges[r][1] - ranges[r][0] > slot_cap:
            raise _lib.CapacityError("a rank emitted more slots than its exchange buffer holds")
        ops.emit(prefixes[r], ranges[r][0])
        plan = exchange_plan(ranges, n_global, p)
        send_chunks, send_sizes = [], []
        for q in range(p):
            first, count = plan[r][q]
            send_sizes.append(count)
            if count:
                send_chunks.append(ops.gather(first, count).t().contiguous())
        recv_sizes = [plan[q][r][1] for q in range(p)]
        send = (torch.cat(send_chunks) if send_chunks else
                torch.empty((0, 5), dtype=torch.float32)).to(dev)
        recv = torch.empty((sum(recv_sizes), 5), dtype=torch.float32, device=dev)
        dist.all_to_all_single(recv, send, output_split_sizes=recv_sizes,
                               input_split_sizes=send_sizes, group=group)
        assert recv.shape[0] == n_local
        ops.set_states(recv.t().contiguous())
    est, ess, res, occ = ops.outputs()
    return est, ess, res, int(np.sum(occ))
