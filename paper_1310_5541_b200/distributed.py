"""Particle-sharded giant filter (BASELINE config 5; new — the reference is
single-process).

One filter of N particles is split across the ranks of a torch.distributed
group (one process per GPU, NCCL over NVLink): rank r holds the global
particles [r n, (r+1) n) and owns the output slots [r n, (r+1) n). Per frame
the ranks exchange exactly what the algorithm needs, with fixed-size
stream-ordered collectives and no host synchronisation (pcs_shard.cuh):

  1. all-reduce MAX of the occupied-cell bounding boxes (5 int64);
  2. all-reduce SUM of the per-cell accumulators over that window, carried as
     int64 limbs of the exact int128 sums in a fixed wcap-cell buffer —
     integer addition is associative, so the dummies are bit-identical for
     every rank count;
  3. every rank runs the same cell / bins stage (dummies, likelihood per
     occupied cell, normaliser, estimate, ESS, resampling decision);
  4. all-gather of the ranks' exact cumulative-weight totals (u128 as three
     42-bit limbs); every rank derives every rank's slot range on the device
     (distributed systematic resampling, monotone ancestors);
  5. each rank emits the ancestors of its own slot range: slots it owns keep
     their ancestors in place (the next frame gathers them directly); only
     the boundary slots owned by rank r-1 / r+1 travel, as states, in fixed
     bcap-slot buffers (grouped send / recv with the two neighbours).

ESS-threshold resampling (``threshold_fraction < 1``, filtering.py:169-171)
adds, between 3 and 4, the per-particle finish of frames whose particles
carry prior weights: all-reduce MAX of the max log-weight, SUM of the exact
normaliser, SUM of the exact estimate / ESS numerators with MAX of the weight
range; then every rank takes the same decision. Frames without prior weights
pass neutral values through the same fixed-size collectives, so the host
never needs to know which kind of frame it is.

Multinomial resampling (filtering.py:96-97,100) replaces 5: the ancestors
are not monotone, so each rank routes its slots to the rank whose part of
the global cdf holds their Philox point (the cdf's values at the rank
boundaries follow from the gathered totals), requests the states of the
remote ancestors (all-to-all of slot offsets, ``bcap`` per rank pair) and
receives them (all-to-all of states).

Philox counters use the global particle index, so the random draws — and
therefore every result — are the same for any number of ranks as for one GPU.
Capacity limits (window, boundary size) are evaluated identically on every
rank; all flags are all-reduced at the end so every rank raises the same
error.

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
    """One rank's compute for the sharded step (see DeviceShardOps). Every
    method returns / takes tensors on the ops' device; nothing synchronises
    the host until flags() / outputs()."""

    def begin(self, cfg, height, width, rank, world, n_global, wcap, bcap, seed):
        raise NotImplementedError

    def step1(self, frame, k):
        """propagate + exact local cell sums -> box int64[5] (MAX-reducible)"""
        raise NotImplementedError

    def export(self, box):
        """window cells of the reduced box -> limbs int64[wcap * 16] (SUM-reducible)"""
        raise NotImplementedError

    def import_bins(self, box, limbs):
        raise NotImplementedError

    def total(self):
        """-> int64[3]: the rank's exact cumulative weight (42-bit limbs)"""
        raise NotImplementedError

    def emit(self, totals):
        """gathered totals int64[world * 3] -> (send_prev, send_next) float32[5 bcap + 1]"""
        raise NotImplementedError

    def unpack(self, recv_prev, recv_next):
        raise NotImplementedError

    def prior(self, stage, red=None, red_mm=None):
        """ESS-threshold frames with prior weights: stage 0 -> (max int64[1], None)
        (MAX), 1 -> (normaliser limbs int64[3], None) (SUM), 2 -> (numerator
        limbs int64[18] (SUM), range int64[2] (MAX)), 3 finalises (-> None)"""
        raise NotImplementedError

    def route(self, totals):
        """multinomial: gathered totals -> requests int32[world * (1 + bcap)]"""
        raise NotImplementedError

    def serve(self, req_in):
        """multinomial: received requests -> answers float32[world * 5 * bcap]"""
        raise NotImplementedError

    def install(self, resp_in):
        raise NotImplementedError

    def flags(self):
        """-> PCS_FLAG_* of this rank (host int; synchronises)"""
        raise NotImplementedError

    def outputs(self):
        """-> (estimates (K,5), ess (K,), resampled (K,), occupied (K,)) host arrays"""
        raise NotImplementedError


class DeviceShardOps(ShardOps):
    """Product implementation: the rank's GPU through the C ABI (pcs_shard_*)."""

    def __init__(self, n_frames, ctx=None):
        self.n_frames = n_frames
        self.ctx = ctx if ctx is not None else _lib.ctx()   # pcs_ctx handle (one per rank)

    def begin(self, cfg, height, width, rank, world, n_global, wcap, bcap, seed):
        self.dev = _lib.device()
        dev = self.dev
        res = cfg.resampling
        self.multi = res.scheme == "multinomial"
        self.pout = [torch.empty(n, dtype=torch.int64, device=dev) for n in (1, 3, 18)]
        self.pmm = torch.empty(2, dtype=torch.int64, device=dev)
        if self.multi:
            self.req = torch.empty(world * (1 + bcap), dtype=torch.int32, device=dev)
            self.resp = torch.zeros(world * 5 * bcap, dtype=torch.float32, device=dev)
        self.est = torch.empty((self.n_frames, 5), dtype=torch.float64, device=dev)
        self.ess = torch.empty(self.n_frames, dtype=torch.float64, device=dev)
        self.res = torch.empty(self.n_frames, dtype=torch.uint8, device=dev)
        self.occ = torch.empty(self.n_frames, dtype=torch.int64, device=dev)
        self.box = torch.empty(5, dtype=torch.int64, device=dev)
        self.limbs = torch.empty(wcap * LIMBS, dtype=torch.int64, device=dev)
        self.tot = torch.empty(3, dtype=torch.int64, device=dev)
        self.send = [torch.zeros(5 * bcap + 1, dtype=torch.float32, device=dev) for _ in range(2)]
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
        c.threshold_fraction = res.threshold_fraction
        c.scheme = 1 if self.multi else 0
        c.weighted_com = 1 if getattr(cfg, "weighted_com", False) else 0
        _lib.check(_lib.lib().pcs_shard_begin(self.ctx, ctypes.byref(c), height, width, rank,
                                              world, n_global, wcap, bcap, _lib.stream()),
                   "pcs_shard_begin")

    def step1(self, frame, k):
        _lib.check(_lib.lib().pcs_shard_step1(
            self.ctx, _lib.ptr(frame), k, _lib.ptr(self.est[k:]), _lib.ptr(self.ess[k:]),
            _lib.ptr(self.res[k:]), _lib.ptr(self.occ[k:]), _lib.ptr(self.box), _lib.stream()),
            "pcs_shard_step1")
        return self.box

    def export(self, box):
        _lib.check(_lib.lib().pcs_shard_export(self.ctx, _lib.ptr(box), _lib.ptr(self.limbs),
                                               _lib.stream()), "pcs_shard_export")
        return self.limbs

    def import_bins(self, box, limbs):
        _lib.check(_lib.lib().pcs_shard_import_bins(self.ctx, _lib.ptr(box), _lib.ptr(limbs),
                                                    _lib.stream()), "pcs_shard_import_bins")

    def total(self):
        _lib.check(_lib.lib().pcs_shard_total(self.ctx, _lib.ptr(self.tot), _lib.stream()),
                   "pcs_shard_total")
        return self.tot

    def emit(self, totals):
        _lib.check(_lib.lib().pcs_shard_emit(self.ctx, _lib.ptr(totals), _lib.ptr(self.send[0]),
                                             _lib.ptr(self.send[1]), _lib.stream()),
                   "pcs_shard_emit")
        return self.send[0], self.send[1]

    def unpack(self, recv_prev, recv_next):
        _lib.check(_lib.lib().pcs_shard_unpack(self.ctx, _lib.ptr(recv_prev), _lib.ptr(recv_next),
                                               _lib.stream()), "pcs_shard_unpack")

    def prior(self, stage, red=None, red_mm=None):
        out = self.pout[stage] if stage < 3 else None
        mm = self.pmm if stage == 2 else None
        _lib.check(_lib.lib().pcs_shard_prior(
            self.ctx, stage, None if red is None else _lib.ptr(red),
            None if red_mm is None else _lib.ptr(red_mm), None if out is None else _lib.ptr(out),
            None if mm is None else _lib.ptr(mm), _lib.stream()), "pcs_shard_prior")
        return out, mm

    def route(self, totals):
        _lib.check(_lib.lib().pcs_shard_route(self.ctx, _lib.ptr(totals), _lib.ptr(self.req),
                                              _lib.stream()), "pcs_shard_route")
        return self.req

    def serve(self, req_in):
        _lib.check(_lib.lib().pcs_shard_serve(self.ctx, _lib.ptr(req_in), _lib.ptr(self.resp),
                                              _lib.stream()), "pcs_shard_serve")
        return self.resp

    def install(self, resp_in):
        _lib.check(_lib.lib().pcs_shard_install(self.ctx, _lib.ptr(resp_in), _lib.stream()),
                   "pcs_shard_install")

    def flags(self):
        out = _lib.PcsTrackResult()
        rc = _lib.lib().pcs_track_end(self.ctx, ctypes.byref(out), _lib.stream())
        if rc not in (0, _lib.E_CAPACITY):
            _lib.check(rc, "pcs_track_end")
        return int(out.flags), int(out.first_bad_frame)

    def outputs(self):
        torch.cuda.synchronize()
        return (self.est.cpu().numpy(), self.ess.cpu().numpy(),
                self.res.cpu().numpy().astype(bool), self.occ.cpu().numpy())


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


def _exchange(send_prev, send_next, rank, world, group):
    """Grouped send / receive of the boundary buffers with the two neighbours
    (fixed sizes; an edge rank's missing neighbour contributes an empty buffer)."""
    recv_prev = torch.zeros_like(send_prev)
    recv_next = torch.zeros_like(send_next)
    ops = []
    if rank > 0:
        ops += [dist.P2POp(dist.isend, send_prev, rank - 1, group),
                dist.P2POp(dist.irecv, recv_prev, rank - 1, group)]
    if rank < world - 1:
        ops += [dist.P2POp(dist.isend, send_next, rank + 1, group),
                dist.P2POp(dist.irecv, recv_next, rank + 1, group)]
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    return recv_prev, recv_next


def _on(t, dev):
    return t if t.device == dev else t.to(dev)


def default_bcap(n_local, world, multinomial):
    """Exchange capacity: boundary slots per neighbour (systematic: the
    weight-share imbalance between neighbouring ranks), or requests per rank
    pair (multinomial: each rank's slots draw ~n_local / world ancestors from
    every rank; 1.5x that plus a margin)."""
    if multinomial:
        return max(1, min(n_local, max(4096, (3 * n_local) // (2 * world) + 1024)))
    return max(1, min(n_local, max(4096, n_local // 4)))


def _all_reduce(t, op, dev, group):
    c = _on(t, dev)
    dist.all_reduce(c, op=op, group=group)
    return _on(c, t.device)


def _all_to_all(t, dev, group):
    c = _on(t, dev)
    out = torch.empty_like(c)
    dist.all_to_all_single(out, c, group=group)
    return _on(out, t.device)


def sharded_pcsir_track(frames, cfg, seed, ops, group=None, wcap=1 << 16, bcap=None,
                        comm_device=None):
    """Run pcSIR over the ranks of ``group``; every rank returns the same
    (estimates, ess, resampled, likelihood_evals), equal to the one-GPU
    filter's for any ResampleConfig (ESS threshold, systematic or
    multinomial).

    ``frames``: (K,H,W) float32 tensor on the rank's device (the frames are
    replicated: every rank evaluates the same occupied cells). ``cfg`` is a
    PcFilterConfig with the GLOBAL n_particles (divisible by the world size).
    ``wcap``: cells of the limb window; ``bcap``: boundary slots exchanged
    with each neighbour per frame (systematic) or requests per rank pair
    (multinomial); default ``default_bcap``."""
    r_cfg = cfg.resampling
    cond = r_cfg.threshold_fraction < 1.0
    multi = r_cfg.scheme == "multinomial"
    p = dist.get_world_size(group)
    r = dist.get_rank(group)
    n_global = cfg.n_particles
    if n_global % p:
        raise ValueError("n_particles must be divisible by the number of ranks")
    n_local = n_global // p
    bcap = int(bcap) if bcap else default_bcap(n_local, p, multi)
    from dataclasses import replace
    local_cfg = replace(cfg, n_particles=n_local)
    k_frames, h, w = frames.shape
    ops.begin(local_cfg, h, w, r, p, n_global, int(wcap), bcap, seed)
    dev = comm_device if comm_device is not None else (
        torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl"
        else torch.device("cpu"))
    MAX, SUM = dist.ReduceOp.MAX, dist.ReduceOp.SUM
    for k in range(k_frames):
        box = _all_reduce(ops.step1(frames[k], k), MAX, dev, group)
        limbs = _all_reduce(ops.export(box), SUM, dev, group)
        ops.import_bins(box, limbs)
        if cond:   # frames whose particles carry prior weights finish per particle
            mx, _ = ops.prior(0)
            s3, _ = ops.prior(1, _all_reduce(mx, MAX, dev, group))
            st, mm = ops.prior(2, _all_reduce(s3, SUM, dev, group))
            ops.prior(3, _all_reduce(st, SUM, dev, group), _all_reduce(mm, MAX, dev, group))
        tot = ops.total()
        parts = [torch.empty_like(_on(tot, dev)) for _ in range(p)]
        dist.all_gather(parts, _on(tot, dev), group=group)
        totals = _on(torch.cat(parts), tot.device)
        if multi:
            req_in = _all_to_all(ops.route(totals), dev, group)
            ops.install(_all_to_all(ops.serve(req_in), dev, group))
        else:
            send_prev, send_next = ops.emit(totals)
            rp, rn = _exchange(_on(send_prev, dev), _on(send_next, dev), r, p, group)
            ops.unpack(_on(rp, send_prev.device), _on(rn, send_next.device))
    flags, first_bad = ops.flags()
    ft = torch.tensor([flags, -first_bad if first_bad >= 0 else -(1 << 40)], dtype=torch.int64,
                      device=dev)
    dist.all_reduce(ft, op=dist.ReduceOp.MAX, group=group)   # every rank raises the same error
    flags = int(ft[0].item())
    if flags & _lib.FLAG_CAPACITY:
        raise _lib.CapacityError("the sharded filter exceeded its exchange capacity (limb window "
                                 "or boundary buffer); raise wcap / bcap")
    if flags & _lib.FLAG_NONFINITE:
        raise ValueError("likelihood values must be finite and >= 0")
    if flags & _lib.FLAG_DEGENERATE:
        from .filtering import DegenerateWeightsError
        raise DegenerateWeightsError("all importance weights vanished",
                                     frame_index=int(-ft[1].item()))
    est, ess, res, occ = ops.outputs()
    return est, ess, res, int(np.sum(occ))
