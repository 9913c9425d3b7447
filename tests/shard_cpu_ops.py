"""CPU stand-in for one rank's device compute in the sharded filter
(TEST INFRASTRUCTURE: lets the gloo tests exercise the real orchestration in
paper_1310_5541_b200.distributed — collectives, limb all-reduce, slot ranges,
exchange plan — without a GPU). Arithmetic follows the canonical conventions
(exact integer sums, exact prefix) through the oracle's C helpers."""

import math

import numpy as np
import torch

from oracle import pcsir_oracle as orc
from paper_1310_5541_b200 import distributed as D

M42 = (1 << 42) - 1


def _fixed(v32, F):
    """round(v * 2^F) for float32 values, as Python ints (oracle C)."""
    v = np.ascontiguousarray(v32, dtype=np.float32)
    out = np.empty(2 * v.size, dtype=np.uint64)
    orc.lib().orc_fixed_f32(orc._p(v), v.size, F, orc._p(out))
    res = []
    for q in range(v.size):
        u = (int(out[2 * q + 1]) << 64) | int(out[2 * q])
        if u >= 1 << 127:
            u -= 1 << 128
        res.append(u)
    return res


def _round_fixed64(x, F):
    return int(round(math.ldexp(x, F)))


def _limbs(v):
    """three 42-bit limbs (the top one signed) of an exact integer"""
    return [v & M42, (v >> 42) & M42, v >> 84]


def _unlimbs(L):
    return int(L[0]) + (int(L[1]) << 42) + (int(L[2]) << 84)


def _ordered(x):
    """order-preserving int64 of a float64 (MAX-reducible)"""
    b = int(np.array([x], dtype=np.float64).view(np.int64)[0])
    return b if b >= 0 else b ^ 0x7FFFFFFFFFFFFFFF


def _unordered(b):
    b = b if b >= 0 else b ^ 0x7FFFFFFFFFFFFFFF
    return float(np.array([b], dtype=np.int64).view(np.float64)[0])


def _bits(w32):
    return int(np.array([w32], dtype=np.float32).view(np.uint32)[0])


class CpuShardOps(D.ShardOps):
    """CPU mirror of DeviceShardOps (pcs_shard.cuh): same buffers (box,
    fixed-size limbs, 42-bit total limbs, boundary buffers with the count in
    the last float), same ranges / capacity checks, canonical arithmetic."""

    def __init__(self, n_frames, frames, sigma_psf=1.5, bg=10.0, sigma_xi=10.0, hw=5):
        self.n_frames = n_frames
        self.frames = frames
        self.spot = (sigma_psf, bg, hw, sigma_xi)

    def begin(self, cfg, height, width, rank, world, n_global, wcap, bcap, seed):
        self.cfg = cfg
        self.thresh = cfg.resampling.threshold_fraction * n_global
        self.multi = cfg.resampling.scheme == "multinomial"
        self.extra = world * bcap if self.multi else 2 * bcap
        self.prior_next = False   # the next frame's particles carry prior weights
        self.wprev = None
        self.n = cfg.n_particles
        self.rank, self.world = rank, world
        self.idx_off = rank * self.n
        self.n_global = n_global
        self.wcap, self.bcap = wcap, bcap
        self.seed = seed
        self.flag = 0
        g = cfg.grid
        self.grid = (g.origin_x, g.origin_y, g.cell_width, g.cell_height, g.n_cols, g.n_rows)
        c = cfg.init.center.as_array()
        z = orc.init_normals(seed, self.n, offset=self.idx_off)
        s = np.zeros((5, self.n + self.extra), dtype=np.float64)
        s[:, :self.n] = np.tile(c, (self.n, 1)).T
        s[0, :self.n] = c[0] + cfg.init.sigma * z[0]
        s[1, :self.n] = c[1] + cfg.init.sigma * z[1]
        self.soa = s.astype(np.float32)
        self.anc = np.arange(self.n)
        self.est = np.zeros((self.n_frames, 5))
        self.ess = np.zeros(self.n_frames)
        self.res = np.zeros(self.n_frames, dtype=bool)
        self.occ = np.zeros(self.n_frames, dtype=np.int64)
        self.k = 0

    def step1(self, frame, k):
        self.k = k
        self.pc_prior = self.prior_next
        d = self.cfg.dynamics
        src = np.ascontiguousarray(self.soa[:, self.anc])
        z = orc.propagate_normals(self.seed, k, self.n, offset=self.idx_off).astype(np.float32)
        self.prop = orc.propagate_f32(src, z, d.sigma_pos, d.sigma_vel, d.sigma_int, d.dt)
        ix, iy = orc.cell_indices(self.prop[0].astype(np.float64), self.prop[1].astype(np.float64),
                                  self.grid)
        self.flat = iy * self.grid[4] + ix
        self.table = {}
        fx = [_fixed(self.prop[c], 40) for c in range(5)]
        for i, f in enumerate(self.flat.tolist()):
            e = self.table.setdefault(f, [0, 0, 0, 0, 0, 0])
            e[0] += 1
            for c in range(5):
                e[1 + c] += fx[c][i]
        keys = np.array(list(self.table))
        ncol = self.grid[4]
        return torch.tensor([-int((keys % ncol).min()), int((keys % ncol).max()),
                             -int((keys // ncol).min()), int((keys // ncol).max()), len(keys)],
                            dtype=torch.int64)

    def _window(self, box):
        b = box.tolist()
        x0, y0 = -b[0], -b[2]
        nx, ny = b[1] - x0 + 1, b[3] - y0 + 1
        return x0, y0, nx, ny, nx >= 1 and ny >= 1 and nx * ny <= self.wcap

    def export(self, box):
        x0, y0, nx, ny, ok = self._window(box)
        limbs = np.zeros((self.wcap, D.LIMBS), dtype=np.int64)
        if not ok:
            self.flag |= 4
            return torch.from_numpy(limbs.reshape(-1))
        ncol = self.grid[4]
        for f, e in self.table.items():
            q = (f // ncol - y0) * nx + (f % ncol - x0)
            limbs[q, 0] = e[0]
            for c in range(5):
                v = e[1 + c]
                limbs[q, 1 + 3 * c] = v & M42
                limbs[q, 2 + 3 * c] = (v >> 42) & M42
                limbs[q, 3 + 3 * c] = v >> 84
        self.table = {}
        return torch.from_numpy(limbs.reshape(-1))

    def import_bins(self, box, limbs):
        x0, y0, nx, ny, ok = self._window(box)
        if not ok:
            self.do_res = self.pc_prior = self.prior_next = False
            return
        ncol = self.grid[4]
        L = limbs.numpy().reshape(self.wcap, D.LIMBS)[: nx * ny]
        cells = {}
        for q in np.flatnonzero(L[:, 0]):
            f = (y0 + q // nx) * ncol + (x0 + q % nx)
            sums = [int(L[q, 1 + 3 * c]) + (int(L[q, 2 + 3 * c]) << 42) + (int(L[q, 3 + 3 * c]) << 84)
                    for c in range(5)]
            cells[int(f)] = (int(L[q, 0]), sums)
        sp, bg, hw, sxi = self.spot
        pix = np.asarray(self.frames[self.k], dtype=np.float32).astype(np.float64)
        fl = sorted(cells)
        dummies = np.empty((5, len(fl)), dtype=np.float32)
        for b, f in enumerate(fl):
            cnt, sums = cells[f]
            for c in range(5):
                dummies[c, b] = np.float32(math.ldexp(float(sums[c]) / cnt, -40))
        dd = dummies.astype(np.float64)
        ll = orc.loglik_gauss(pix, dd[0], dd[1], dd[4], sp, bg, hw, sxi)
        self.occ[self.k] = len(fl)
        if self.pc_prior:   # finished per particle (prior)
            self.cell_ll = {f: float(ll[b]) for b, f in enumerate(fl)}
            return
        m = ll.max()
        S = sum(cells[f][0] * _round_fixed64(math.exp(ll[b] - m), 95) for b, f in enumerate(fl))
        Sf = math.ldexp(float(S), -95)
        self.wmap = {}
        est = [0] * 5
        w2 = 0
        for b, f in enumerate(fl):
            w = np.float32(math.exp(ll[b] - m) / Sf)
            self.wmap[f] = w
            wq = _fixed(np.array([w]), 62)[0]
            for c in range(5):
                est[c] += wq * cells[f][1][c]
            w2 += cells[f][0] * _round_fixed64(float(w) * float(w), 120)
        k = self.k
        ws = [_bits(w) for w in self.wmap.values()]
        self._decide(est, w2, min(ws) != max(ws))
        self.w = np.array([self.wmap[f] for f in self.flat.tolist()], dtype=np.float32)

    def _decide(self, est, w2, unequal):
        k = self.k
        self.est[k] = [math.ldexp(float(v), -102) for v in est]
        self.ess[k] = 1.0 / math.ldexp(float(w2), -120)
        self.do_res = self.ess[k] < self.thresh
        self.res[k] = self.do_res
        self.prior_next = (not self.do_res) and unequal
        self.u = orc.resample_u(self.seed, k)

    def prior(self, stage, red=None, red_mm=None):
        """per-particle finish of a frame with prior weights (neutral values otherwise)"""
        on = self.pc_prior
        if stage == 0:
            v = -(1 << 63)
            if on:
                self.pll = np.log(self.wprev.astype(np.float64)) + np.array(
                    [self.cell_ll[f] for f in self.flat.tolist()])
                v = _ordered(float(self.pll.max()))
            return torch.tensor([v], dtype=torch.int64), None
        if stage == 1:
            S = 0
            if on:
                m = _unordered(int(red[0]))
                self.ex = np.exp(self.pll - m)
                S = sum(_round_fixed64(float(e), 95) for e in self.ex)
            return torch.tensor(_limbs(S), dtype=torch.int64), None
        if stage == 2:
            out = [0] * 18
            mm = [-0xFFFFFFFF, 0]
            if on:
                Sf = math.ldexp(float(_unlimbs(red.tolist())), -95)
                self.w = (self.ex / Sf).astype(np.float32)
                wq = _fixed(self.w, 62)
                fx = [_fixed(self.prop[c], 40) for c in range(5)]
                est = [sum(a * b for a, b in zip(wq, fx[c])) for c in range(5)]
                w2 = sum(_round_fixed64(float(w) * float(w), 120) for w in self.w)
                out = sum((_limbs(v) for v in est + [w2]), [])
                bits = self.w.view(np.uint32)
                mm = [-int(bits.min()), int(bits.max())]
            return (torch.tensor(out, dtype=torch.int64), torch.tensor(mm, dtype=torch.int64))
        if on:
            L = red.tolist()
            est = [_unlimbs(L[3 * c:3 * c + 3]) for c in range(5)]
            w2 = _unlimbs(L[15:18])
            self._decide(est, w2, -int(red_mm[0]) != int(red_mm[1]))
        return None, None

    def total(self):
        out = np.zeros(3, dtype=np.int64)
        if self.do_res:
            wx = _fixed(self.w, 120)
            self.incl = np.cumsum(np.array(wx, dtype=object))
            t = int(self.incl[-1])
            out[:] = [t & M42, (t >> 42) & M42, t >> 84]
        return torch.from_numpy(out)

    def _buffers(self):
        return [np.zeros(5 * self.bcap + 1, dtype=np.float32) for _ in range(2)]

    @staticmethod
    def _set_count(buf, cnt):
        buf[-1:] = np.array([cnt], dtype=np.int32).view(np.float32)

    def emit(self, totals):
        bufs = self._buffers()
        n, r, p, ng, bcap = self.n, self.rank, self.world, self.n_global, self.bcap
        if not self.do_res or self.flag & 4:
            self._identity()
            self.recv_counts = (0, 0)
            return torch.from_numpy(bufs[0]), torch.from_numpy(bufs[1])
        T = totals.numpy().reshape(p, 3)
        tots = [int(T[q, 0]) + (int(T[q, 1]) << 42) + (int(T[q, 2]) << 84) for q in range(p)]
        u = self.u
        # every rank's range (k_shard_ranges), the same capacity checks
        lo, pre, ranges, prefixes = 0, 0, [], []
        for q in range(p):
            hi = ng if q == p - 1 else D.first_slot(D.cdf_value(pre + tots[q]), u, ng)
            own0, own1 = q * n, (q + 1) * n
            if (lo < own0 - n or hi > own1 + n or hi - lo > n + 2 * bcap
                    or max(0, min(hi, own0) - lo) > bcap or max(0, hi - max(lo, own1)) > bcap):
                self.flag |= 4
            ranges.append((lo, hi))
            prefixes.append(pre)
            pre += tots[q]
            lo = hi
        if self.flag & 4:
            self._identity()
            self.recv_counts = (0, 0)
            return torch.from_numpy(bufs[0]), torch.from_numpy(bufs[1])
        lo_r, hi_r = ranges[r]
        # ancestors of slots [lo_r, hi_r) from this rank's exact prefixes
        anc_out = []
        j = lo_r
        for i in range(n):
            gi = self.idx_off + i
            jend = ng if gi == ng - 1 else D.first_slot(
                D.cdf_value(prefixes[r] + int(self.incl[i])), u, ng)
            anc_out.extend([i] * (jend - j))
            j = max(j, jend)
        assert len(anc_out) == hi_r - lo_r
        own0, own1 = r * n, (r + 1) * n
        anc = np.full(n, -1, dtype=np.int64)
        sp, sn = 0, 0
        for s_, src in enumerate(anc_out):
            jj = lo_r + s_
            if jj < own0:
                bufs[0][np.arange(5) * bcap + (jj - lo_r)] = self.prop[:, src]
                sp += 1
            elif jj >= own1:
                bufs[1][np.arange(5) * bcap + (jj - own1)] = self.prop[:, src]
                sn += 1
            else:
                anc[jj - own0] = src
        self._set_count(bufs[0], sp)
        self._set_count(bufs[1], sn)
        self.anc = anc
        hi_prev = ranges[r - 1][1] if r > 0 else own0
        lo_next = ranges[r + 1][0] if r < p - 1 else own1
        self.recv_counts = (max(0, hi_prev - own0), max(0, own1 - lo_next))
        self.next_soa = self._extended(self.prop)
        return torch.from_numpy(bufs[0]), torch.from_numpy(bufs[1])

    def _extended(self, prop):
        s = np.zeros((5, self.n + self.extra), dtype=np.float32)
        s[:, :self.n] = prop
        return s

    def _identity(self):
        """no resampling: identity ancestors; unequal weights go to the next frame"""
        self.anc = np.arange(self.n)
        self.next_soa = self._extended(self.prop)
        if self.prior_next and not self.flag & 4:
            self.wprev = self.w.copy()

    # ---- multinomial ----
    def _points(self):
        return orc.multinomial_points(self.seed, self.k, self.n_global)

    def route(self, totals):
        n, r, p, bcap = self.n, self.rank, self.world, self.bcap
        req = np.zeros((p, 1 + bcap), dtype=np.int32)
        self.sent = [0] * p
        if not self.do_res or self.flag & 4:
            self._identity()
            return torch.from_numpy(req.reshape(-1))
        T = totals.numpy().reshape(p, 3)
        tots = [_unlimbs(T[q]) for q in range(p)]
        pre = [0]
        for q in range(p):
            pre.append(pre[-1] + tots[q])
        bnd = [D.cdf_value(pre[q]) for q in range(p)]
        wx = _fixed(self.w, 120)
        cdf, run = [], pre[r]
        for i in range(n):
            run += wx[i]
            cdf.append(1.0 if self.idx_off + i == self.n_global - 1 else D.cdf_value(run))
        self.cdf = np.array(cdf)
        pts = self._points()[self.idx_off:self.idx_off + n]
        anc = np.empty(n, dtype=np.int64)
        for jl in range(n):
            q = sum(1 for b in range(1, p) if bnd[b] <= pts[jl])
            if q == r:
                anc[jl] = min(int(np.searchsorted(self.cdf, pts[jl], side="right")), n - 1)
            elif self.sent[q] < bcap:
                req[q, 1 + self.sent[q]] = jl
                anc[jl] = n + q * bcap + self.sent[q]
                self.sent[q] += 1
            else:
                self.flag |= 4
        req[:, 0] = self.sent
        self.anc = anc
        self.next_soa = self._extended(self.prop)
        return torch.from_numpy(req.reshape(-1))

    def serve(self, req_in):
        n, r, p, bcap = self.n, self.rank, self.world, self.bcap
        resp = np.zeros((p, 5, bcap), dtype=np.float32)
        if self.do_res and not self.flag & 4:
            R = req_in.numpy().reshape(p, 1 + bcap)
            pts = self._points()
            for q in range(p):
                if q == r:
                    continue
                for s_ in range(int(R[q, 0])):
                    i = min(int(np.searchsorted(self.cdf, pts[q * n + int(R[q, 1 + s_])],
                                                side="right")), n - 1)
                    resp[q, :, s_] = self.prop[:, i]
        return torch.from_numpy(resp.reshape(-1))

    def install(self, resp_in):
        n, r, p, bcap = self.n, self.rank, self.world, self.bcap
        if self.do_res and not self.flag & 4:
            R = resp_in.numpy().reshape(p, 5, bcap)
            for q in range(p):
                if q != r:
                    c = self.sent[q]
                    self.next_soa[:, n + q * bcap:n + q * bcap + c] = R[q, :, :c]
        self.soa = self.next_soa

    def unpack(self, recv_prev, recv_next):
        n, bcap = self.n, self.bcap
        cp, cn = self.recv_counts
        rp, rn = recv_prev.numpy(), recv_next.numpy()
        for q in range(cp):
            self.next_soa[:, n + q] = rp[np.arange(5) * bcap + q]
            self.anc[q] = n + q
        for q in range(cn):
            self.next_soa[:, n + bcap + q] = rn[np.arange(5) * bcap + q]
            self.anc[n - cn + q] = n + bcap + q
        assert (self.anc >= 0).all()
        self.soa = self.next_soa

    def flags(self):
        return self.flag, -1

    def outputs(self):
        return self.est, self.ess, self.res, self.occ
