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


class CpuShardOps(D.ShardOps):
    def __init__(self, n_frames, frames, sigma_psf=1.5, bg=10.0, sigma_xi=10.0, hw=5):
        self.n_frames = n_frames
        self.frames = frames
        self.spot = (sigma_psf, bg, hw, sigma_xi)

    def begin(self, cfg, height, width, idx_off, n_global, slot_cap, seed):
        self.cfg = cfg
        self.n = cfg.n_particles
        self.idx_off = idx_off
        self.n_global = n_global
        self.seed = seed
        g = cfg.grid
        self.grid = (g.origin_x, g.origin_y, g.cell_width, g.cell_height, g.n_cols, g.n_rows)
        c = cfg.init.center.as_array()
        z = orc.init_normals(seed, self.n, offset=idx_off)
        s = np.tile(c, (self.n, 1)).T.copy()
        s[0] = c[0] + cfg.init.sigma * z[0]
        s[1] = c[1] + cfg.init.sigma * z[1]
        self.soa = s.astype(np.float32)
        self.anc = np.arange(self.n)
        self.est = np.zeros((self.n_frames, 5))
        self.ess = np.zeros(self.n_frames)
        self.res = np.zeros(self.n_frames, dtype=bool)
        self.occ = np.zeros(self.n_frames, dtype=np.int64)
        self.k = 0

    def step1(self, frame, k):
        self.k = k
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
        return [int((keys % ncol).min()), int((keys % ncol).max()), int((keys // ncol).min()),
                int((keys // ncol).max())], len(keys)

    def export(self, window):
        x0, y0, nx, ny = window
        ncol = self.grid[4]
        limbs = np.zeros((nx * ny, D.LIMBS), dtype=np.int64)
        for f, e in self.table.items():
            q = (f // ncol - y0) * nx + (f % ncol - x0)
            limbs[q, 0] = e[0]
            for c in range(5):
                v = e[1 + c]
                limbs[q, 1 + 3 * c] = v & M42
                limbs[q, 2 + 3 * c] = (v >> 42) & M42
                limbs[q, 3 + 3 * c] = v >> 84
        self.table = {}
        return torch.from_numpy(limbs)

    def import_bins(self, window, limbs):
        x0, y0, nx, ny = window
        ncol = self.grid[4]
        L = limbs.numpy()
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
        self.est[k] = [math.ldexp(float(v), -102) for v in est]
        self.ess[k] = 1.0 / math.ldexp(float(w2), -120)
        self.do_res = self.ess[k] < self.n_global
        self.res[k] = self.do_res
        self.occ[k] = len(fl)

    def scan(self):
        w = np.array([self.wmap[f] for f in self.flat.tolist()], dtype=np.float32)
        wx = _fixed(w, 120)
        self.incl = np.cumsum(np.array(wx, dtype=object))
        return int(self.incl[-1]), bool(self.do_res)

    def emit(self, prefix, slot_lo):
        u = orc.resample_u(self.seed, self.k)
        anc = []
        j = 0 if (self.idx_off == 0) else D.first_slot(D.cdf_value(prefix), u, self.n_global)
        for i in range(self.n):
            gi = self.idx_off + i
            jend = self.n_global if gi == self.n_global - 1 else D.first_slot(
                D.cdf_value(prefix + int(self.incl[i])), u, self.n_global)
            anc.extend([i] * (jend - j))
            j = max(j, jend)
        self.anc_out = np.array(anc, dtype=np.int64)

    def gather(self, first, count):
        return torch.from_numpy(np.ascontiguousarray(self.prop[:, self.anc_out[first:first + count]]))

    def set_states(self, soa):
        self.soa = soa.numpy().astype(np.float32)
        self.anc = np.arange(self.n)

    def advance(self):
        self.soa = self.prop
        self.anc = np.arange(self.n)

    def outputs(self):
        return self.est, self.ess, self.res, self.occ

    def resample_u(self, seed, frame):
        return orc.resample_u(seed, frame)
