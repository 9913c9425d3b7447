// pcs_multi.cuh — batched multi-target pcSIR (config 4; new — the reference
// tracks one spot per filter).
//
// One CTA owns one target for a whole frame and runs the complete pcsir_track
// step (binning.py:175-195 + filtering.py:148-173) for that target with
// block-level synchronisation only:
//   A  gather + propagate + cell index + exact per-cell sums (32-bit shared
//      atomics into a shared-memory sub-window; outliers into a per-target
//      HBM hash table with exact limb reductions)
//   B  occupied cells -> dummies -> likelihood (frame region staged in shared
//      memory) -> exact normaliser -> per-cell weights, estimate, ESS, decision
//   C  exact-prefix systematic resampling over the target's particles (tiles
//      scanned in order inside the CTA; no inter-CTA look-back needed), or the
//      exact cdf and a binary search of the frame's Philox points (multinomial)
// With ESS-threshold resampling a frame that does not resample hands its
// normalised weights to the next one (wprev); that frame's weights are then
// per particle, log w = log w_prev + ll[cell] (binning.py:190-192,
// filtering.py:69,169-171), and phase B finishes it per particle with the
// canonical sums of the single-target kernels (k_pc_prior_ll, k_sir_sum,
// k_sir_stats).
// Target t uses the RNG key seed_t = seed + t*0x9E3779B97F4A7C15 with local
// particle indices, so every target equals a single-target pcsir_track run
// with seed_t bit for bit (tests/test_gpu_multi.py).
#pragma once
#include "pcs_common.cuh"
#include "pcs_fused.cuh"
#include "pcs_lik.cuh"
#include "pcs_state.cuh"
#include "pcs_weights.cuh"

namespace pcs {

// Two CTAs per SM (<= 64 registers, < 113 KB shared memory each): the
// sub-window is 24 x 24 cells (a c4 cloud spans a few pixels; cells outside
// it go to the exact per-target hash), and the phase-A tile, the phase-B
// cell arrays and the phase-C scan buffers share one union.
#ifndef PCS_MT_THREADS
#define PCS_MT_THREADS 512
#endif
constexpr int MT_THREADS = PCS_MT_THREADS;
#ifndef PCS_MT_IPT
#define PCS_MT_IPT 1   // (1 / 2 / 3 particles per thread and tile: c4 11.93 / 12.21 / 13.22 ms)
#endif
constexpr int MT_IPT = PCS_MT_IPT;
constexpr int MT_TILE = MT_THREADS * MT_IPT;   // 512
constexpr int MT_WARPS = MT_THREADS / 32;
constexpr int MT_SIDE = 24;
constexpr int MT_SUBW = MT_SIDE * MT_SIDE;     // sub-window cells (24 x 24)
#ifndef PCS_MT_MARGIN
#define PCS_MT_MARGIN 3
#endif
constexpr int MT_MARGIN = PCS_MT_MARGIN;       // sub-window cells beyond the previous frame's span
#ifndef PCS_MT_PREFETCH
#define PCS_MT_PREFETCH 1
#endif
constexpr int MT_HCAP = 2048;                  // per-target outlier hash capacity
constexpr int MT_MAXM = 2048;                  // occupied cells per target per frame
constexpr int MT_STAGE = 4096;                 // staged frame pixels
#ifndef PCS_MT_CI
#define PCS_MT_CI 11   // (7 / 9 / 11: c4 12.10 / 11.95 / 11.81 ms; 13 would not fit two CTAs per SM)
#endif
constexpr int MT_CI = PCS_MT_CI;                       // phase C: items per thread (odd stride: conflict-free)
constexpr int MT_CT = MT_THREADS * MT_CI;      // phase C: 5632 particles per scan tile
// phase A digit accumulators: one addition per particle of each digit of
// V = round(v 2^40) (|V| < 2^47): bits 0-13, 14-27, 28-41 (< 2^14 each) and
// V >> 42 (signed, |.| <= 2^5), so n <= 2^18 particles per target keep every
// 32-bit accumulator in range
constexpr int MT_MAX_TILES = (1 << 18) / MT_TILE;   // n <= MT_MAX_TILES * MT_TILE = 2^18
constexpr int MT_DIG = 20;          // 5 components x 4 digits
constexpr u64 MT_KEY_STEP = 0x9E3779B97F4A7C15ull;

struct MtTarget {
  double center[2];
  u32 flags;
  int first_bad;
  i64 evals;
  int prior;             // this frame's particles carry prior weights (wprev)
  int span;              // extent (cells) of the previous frame's occupied cells, 0 = unknown
};

struct MtHash {          // one outlier cell
  u32 key;               // flat cell + 1 (0 = empty)
  u32 cnt;
  u64 lim[5][3];         // exact sums as limbs: bits 0-31 and 32-63 (unsigned), the rest
                         // (signed), added with fire-and-forget reductions (tab_add_f32)
  u64 stash;             // phase B -> C: the cell's weight (float bits) or, with prior
                         // weights, its log-likelihood (double bits)
};
// exact int128 sum of component c of an outlier cell
__device__ __forceinline__ i128 mt_hash_sum(const MtHash& h, int c) {
  return (i128)h.lim[c][0] + ((i128)h.lim[c][1] << 32) + ((i128)(long long)h.lim[c][2] << 64);
}
__device__ __forceinline__ void mt_hash_clear(MtHash& h) {
#pragma unroll
  for (int c = 0; c < 5; ++c) h.lim[c][0] = h.lim[c][1] = h.lim[c][2] = 0ull;
}

struct MtParams {
  i64 T, n, ld;          // targets on this rank, particles per target, SoA stride (= T*n)
  i64 H, W;
  Dyn dyn;
  Spot spot;
  Grid grid;
  double inv_lx, inv_ly;
  int pow2;              // grid_pow2 of the grid (cell_axis_hot<true> applies)
  u64 seed;
  i64 tgt_off;           // global index of target 0 of this rank (RNG key)
  u32 frame0;
  int placement;
  float* buf0;
  float* buf1;
  int* anc;
  u32* pslot;
  MtTarget* tgt;
  MtHash* hash;          // [T][MT_HCAP]
  const float* frame;    // current frame
  i64 k;                 // frame index (buffer parity, RNG frame, output row)
  i64 K;                 // output rows per target
  double thresh;         // resample when ESS < thresh (threshold_fraction * n)
  int multinomial;       // resampling scheme (filtering.py:96-100)
  float* wprev;          // [T*n] prior weights (threshold < 1; else null)
  double* ll;            // [T*n] per-particle log w, then exp(log w - m) (prior frames)
  double* cdf;           // [T*n] exact cdf (multinomial; else null)
  double* out_est;       // [T][K][5]
  double* out_ess;       // [T][K]
  unsigned char* out_res;
  i64* out_occ;
};

struct MtSmem {
  // phase A (as k_pc_step1: every in-window particle adds its exact values
  // to the cell's 32-bit digit accumulators with shared atomics; cells at
  // s1_swz positions to spread a cloud over the banks)
  u32 dig[MT_DIG][MT_SUBW];
  u32 acc_cnt[MT_SUBW];
  u128 wfix_sub[MT_SUBW];          // exact cdf weight round(w 2^120) per sub-window cell
                                   // (prior frames: the cell log-likelihood, as double)
  float wsub_f[MT_SUBW];           // normalised weight per sub-window cell (wprev)
  float ref[2 * MT_SIDE + 1];      // sub-window cell edges (x then y; NaN: unusable)
  union {
    struct {                       // phase B: occupied cells, dummies, staged frame
      int occ[MT_MAXM];            // >= 0: sub-window cell, < 0: -(hash slot) - 1
      double ll[MT_MAXM];
      float dpix[MT_STAGE];
    } b;
    struct {                       // phase C: staged cells (then each item's run head,
      u32 cells[MT_CT];            // written over the item's consumed cell), slot stage
      int stage[MT_CT];
    } c;
  } u;
  int scan_tmp[MT_WARPS];
  i128 red[MT_WARPS * 6];
  long long lmax;
  long long plmax;                 // prior frames: max per-particle log w
  int box[4];
  int obox[4];                     // occupied cells' bounds relative to the sub-window origin
  u32 n_occ;
  int fast_delta;
  unsigned wmin, wmax;
  double Sf;
  u128 carry;
  u128 wtot[MT_WARPS];
};

__device__ __forceinline__ u32 mt_hash_slot(u32 key) { return (key * 2654435761u) & (MT_HCAP - 1); }

// slot of outlier cell `flat` (present: it holds a particle of this frame)
__device__ __forceinline__ u32 mt_hash_find(const MtHash* H, u32 flat) {
  const u32 key = flat + 1u;
  u32 s = mt_hash_slot(key);
  for (int probe = 0; probe < MT_HCAP && H[s].key != key; ++probe) s = (s + 1u) & (MT_HCAP - 1);
  return s;
}

// add a particle to the target's outlier hash table: the key by CAS (a plain
// load first finds an existing key without an atomic round trip), the count
// and the exact limbs with fire-and-forget reductions
__device__ __forceinline__ bool mt_hash_add(MtHash* H, u32 flat, const float o[5]) {
  u32 key = flat + 1u;
  u32 s = mt_hash_slot(key);
  for (int probe = 0; probe < MT_HCAP; ++probe) {
    u32 prev = __ldcg(&H[s].key);
    if (prev != key) prev = atomicCAS(&H[s].key, 0u, key);
    if (prev == 0u || prev == key) {
      atomicAdd(&H[s].cnt, 1u);
#pragma unroll
      for (int c = 0; c < 5; ++c) tab_add_f32(&H[s].lim[c][0], o[c]);
      return true;
    }
    s = (s + 1u) & (MT_HCAP - 1);
  }
  return false;
}

// exact int128 value of component c of sub-window cell q (unswizzled index)
__device__ __forceinline__ i128 mt_digits(const u32 (*dig)[MT_SUBW], int c, int q) {
  const int qs = s1_swz(q);
  return (i128)dig[4 * c][qs] + ((i128)dig[4 * c + 1][qs] << 14) + ((i128)dig[4 * c + 2][qs] << 28) +
         ((i128)(int)dig[4 * c + 3][qs] << 42);
}
__device__ __forceinline__ void mt_add(u32 (*dig)[MT_SUBW], int qs, const float (&v)[5]) {
#pragma unroll
  for (int c = 0; c < 5; ++c) {
    const long long V = __float2ll_rn(__fmul_rn(v[c], 1099511627776.0f));
    const u32 lo = (u32)V;
    atomicAdd(&dig[4 * c][qs], lo & 0x3FFFu);
    atomicAdd(&dig[4 * c + 1][qs], (lo >> 14) & 0x3FFFu);
    atomicAdd(&dig[4 * c + 2][qs], (u32)(V >> 28) & 0x3FFFu);
    atomicAdd(&dig[4 * c + 3][qs], (u32)(V >> 42));
  }
}

// GEN: ESS-threshold and / or multinomial resampling compiled in (the
// every-frame systematic configuration runs the instantiation without them)
template <int MAXS, bool GEN>
#ifndef PCS_MT_CTAS
#define PCS_MT_CTAS 2
#endif
__global__ void __launch_bounds__(MT_THREADS, PCS_MT_CTAS) k_mt_frame(MtParams P) {
  extern __shared__ __align__(16) unsigned char mt_raw[];
  MtSmem& sm = *reinterpret_cast<MtSmem*>(mt_raw);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const i64 tg = blockIdx.x;
  MtTarget& TG = P.tgt[tg];
  if (TG.flags & PCS_FLAG_CAPACITY) return;   // this target needs the general path
  const bool prior = GEN && TG.prior != 0;     // (thread 0 rewrites it in phase B)
  const u64 seed_t = P.seed + (u64)(P.tgt_off + tg) * MT_KEY_STEP;
  const i64 n = P.n, ld = P.ld, base_i = tg * n;
  const i64 k = P.k;
  const float* sin = (k & 1) ? P.buf1 : P.buf0;
  float* sout = (k & 1) ? P.buf0 : P.buf1;
  const Grid g = P.grid;
  MtHash* HT = P.hash + tg * MT_HCAP;

  // ---------------- phase A: propagate + exact per-cell sums -------------------
  // A compact cloud (the previous frame's occupied cells span <= side - 4
  // cells) gets a smaller sub-window and `rep` replicas of its accumulators
  // (replica = lane % rep, folded after the particle loop): at 1 px cells a
  // warp's particles share ~10 cells and their shared atomics would
  // serialise on those addresses. The sums are exact integers, so the result
  // does not depend on the choice.
  int side = MT_SIDE, rep = 1;
  {
    const int span = TG.span;
    if (span > 0 && span + MT_MARGIN <= 6) { side = 6; rep = 16; }
    else if (span > 0 && span + MT_MARGIN <= 8) { side = 8; rep = 8; }
    else if (span > 0 && span + MT_MARGIN <= 12) { side = 12; rep = 4; }
  }
  const i64 snx = min((i64)side, g.ncols), sny = min((i64)side, g.nrows);
  const i64 cx = cell_axis_fast((float)TG.center[0], g.ox, g.lx, P.inv_lx, g.ncols);
  const i64 cy = cell_axis_fast((float)TG.center[1], g.oy, g.ly, P.inv_ly, g.nrows);
  const i64 sx0 = min(max(cx - snx / 2, (i64)0), g.ncols - snx);
  const i64 sy0 = min(max(cy - sny / 2, (i64)0), g.nrows - sny);
  for (int q = t; q < MT_SUBW; q += MT_THREADS) {
    sm.acc_cnt[q] = 0;
#pragma unroll
    for (int p = 0; p < MT_DIG; ++p) sm.dig[p][q] = 0;
  }
  const int snxi = (int)snx, snyi = (int)sny;
  // fast_delta: every sub-window edge r is >= 2 l (l < 64), so x - r is exact
  // for every x of the cell (Sterbenz) and needs no TwoSum check (k_pc_step1)
  if (t == 0) sm.fast_delta = (g.lx < 64.0 && g.ly < 64.0) ? 1 : 0;
  __syncthreads();
  for (int q = t; q < snxi + snyi; q += MT_THREADS) {
    bool ok;
    float r = (q < snxi) ? cell_ref32(g.ox, g.lx, sx0 + q, ok)
                         : cell_ref32(g.oy, g.ly, sy0 + (q - snxi), ok);
    sm.ref[q] = ok ? r : __int_as_float(0x7fc00000);
    const double l2 = 2.0 * ((q < snxi) ? g.lx : g.ly);
    if (!ok || !((double)r >= l2)) atomicAnd(&sm.fast_delta, 0);
  }
  const float* refy = sm.ref + snxi;
  // the target's Philox round keys once per CTA (not per particle)
  const PhiloxKey pk = philox_key(seed_t);
  // power-of-two cells and float32-exact origins: the margin-free cell index
  const bool pow2 = P.pow2 != 0;
  const AxisFast axx = make_axis(g.ox, g.lx, P.inv_lx, g.ncols);
  const AxisFast axy = make_axis(g.oy, g.ly, P.inv_ly, g.nrows);
  const u32 ncols32 = (u32)g.ncols;
  const int sx0i = (int)sx0, sy0i = (int)sy0;
  if (t == 0) {
    sm.n_occ = 0;
    sm.lmax = LLONG_MIN;
    sm.plmax = LLONG_MIN;
    sm.wmin = 0xFFFFFFFFu;
    sm.wmax = 0u;
    sm.box[0] = INT_MAX; sm.box[1] = INT_MIN; sm.box[2] = INT_MAX; sm.box[3] = INT_MIN;
    sm.obox[0] = INT_MAX; sm.obox[1] = INT_MIN; sm.obox[2] = INT_MAX; sm.obox[3] = INT_MIN;
  }
  __syncthreads();
  const bool fast_delta = sm.fast_delta != 0;
  const int rstride = snxi * snyi;                  // rep * rstride <= MT_SUBW
  const int roff = (lane & (rep - 1)) * rstride;    // this lane's replica
  bool bad = false, hash_full = false;
  const i64 ntile = ceil_div(n, MT_TILE);
  for (i64 tile = 0; tile < ntile; ++tile) {
    int src_k[MT_IPT];
    float o_k[MT_IPT][5];
#pragma unroll
    for (int it = 0; it < MT_IPT; ++it) {
      i64 j = tile * MT_TILE + (i64)it * MT_THREADS + t;
      src_k[it] = (j < n) ? __ldg(P.anc + base_i + j) : 0;
#if PCS_MT_PREFETCH
      // the next tile's ancestor indices on their way to L1 (the gather below
      // waits on them first)
      if (lane == 0 && j + MT_TILE < n)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(P.anc + base_i + j + MT_TILE));
#endif
    }
#pragma unroll
    for (int it = 0; it < MT_IPT; ++it) {
      i64 j = tile * MT_TILE + (i64)it * MT_THREADS + t;
#pragma unroll
      for (int c = 0; c < 5; ++c)
        o_k[it][c] = (j < n) ? __ldg(sin + c * ld + base_i + src_k[it]) : 0.0f;
    }
#pragma unroll
    for (int it = 0; it < MT_IPT; ++it) {
      i64 j = tile * MT_TILE + (i64)it * MT_THREADS + t;
      if (j >= n) continue;
      float s[5], z[5];
#pragma unroll
      for (int c = 0; c < 5; ++c) s[c] = o_k[it][c];
      philox_normals5k(pk, P.frame0 + (u32)k, (u64)j, z);
      propagate_one(s, z, P.dyn, o_k[it]);
      const float* o = o_k[it];
#pragma unroll
      for (int c = 0; c < 5; ++c) __stcs(sout + c * ld + base_i + j, o[c]);   // (read next frame: > L2)
      if (!(o[0] == o[0]) || !(o[1] == o[1])) bad = true;
      const int ix = pow2 ? cell_axis_hot<true>(o[0], axx) : cell_axis_hot<false>(o[0], axx);
      const int iy = pow2 ? cell_axis_hot<true>(o[1], axy) : cell_axis_hot<false>(o[1], axy);
      const u32 flat = (u32)iy * ncols32 + (u32)ix;
      const int lx = ix - sx0i, ly = iy - sy0i;
      float dx, dy;
      bool dok = false;
      if ((u32)lx < (u32)snxi && (u32)ly < (u32)snyi) {
        if (fast_delta) {   // (CTA-uniform branch)
          dx = __fsub_rn(o[0], sm.ref[lx]);
          dy = __fsub_rn(o[1], refy[ly]);
          dok = true;
        } else {
          dok = delta_exact(o[0], sm.ref[lx], dx) && delta_exact(o[1], refy[ly], dy);
        }
      }
      if (dok && fabsf(o[2]) < 128.0f && fabsf(o[3]) < 128.0f && fabsf(o[4]) < 128.0f) {
        const int q = ly * snxi + lx;
        const int qs = s1_swz(q + roff);
        atomicAdd(&sm.acc_cnt[qs], 1u);
        o_k[it][0] = dx;
        o_k[it][1] = dy;
        mt_add(sm.dig, qs, o_k[it]);
        P.pslot[base_i + j] = (u32)q;                 // phase C: sub-window cell
      } else {
        P.pslot[base_i + j] = 0x80000000u | flat;     // phase C: outlier (hash) cell
        if (!mt_hash_add(HT, flat, o)) hash_full = true;
      }
    }
  }
  __syncthreads();
  if (bad) atomicOr(&TG.flags, (u32)PCS_FLAG_NONFINITE);
  if (hash_full) atomicOr(&TG.flags, (u32)PCS_FLAG_CAPACITY);
  if (rep > 1) {   // fold the replicas into replica 0 (modulo 2^32, as the atomics)
    for (int q = t; q < rstride; q += MT_THREADS) {
      const int q0 = s1_swz(q);
      for (int r = 1; r < rep; ++r) {
        const int qi = s1_swz(q + r * rstride);
        sm.acc_cnt[q0] += sm.acc_cnt[qi];
#pragma unroll
        for (int p = 0; p < MT_DIG; ++p) sm.dig[p][q0] += sm.dig[p][qi];
      }
    }
    __syncthreads();
  }

  // ---------------- phase B: occupied cells, dummies, likelihood ----------------
  {
    int ox0 = INT_MAX, ox1 = INT_MIN, oy0 = INT_MAX, oy1 = INT_MIN;
    for (int q = t; q < (int)(snx * sny); q += MT_THREADS) {
      if (sm.acc_cnt[s1_swz(q)]) {
        u32 idx = atomicAdd(&sm.n_occ, 1u);
        if (idx < (u32)MT_MAXM) sm.u.b.occ[idx] = q;
        const int lx = q % snxi, ly = q / snxi;
        ox0 = min(ox0, lx); ox1 = max(ox1, lx); oy0 = min(oy0, ly); oy1 = max(oy1, ly);
      }
    }
    for (int s = t; s < MT_HCAP; s += MT_THREADS) {
      const u32 key = HT[s].key;
      if (key) {
        u32 idx = atomicAdd(&sm.n_occ, 1u);
        if (idx < (u32)MT_MAXM) sm.u.b.occ[idx] = -s - 1;
        const i64 fl = (i64)(key - 1u);
        const int lx = (int)(fl % g.ncols - sx0), ly = (int)(fl / g.ncols - sy0);
        ox0 = min(ox0, lx); ox1 = max(ox1, lx); oy0 = min(oy0, ly); oy1 = max(oy1, ly);
      }
    }
    if (ox0 <= ox1) {
      atomicMin(&sm.obox[0], ox0); atomicMax(&sm.obox[1], ox1);
      atomicMin(&sm.obox[2], oy0); atomicMax(&sm.obox[3], oy1);
    }
  }
  __syncthreads();
  const int M = (int)min(sm.n_occ, (u32)MT_MAXM);
  if (sm.n_occ > (u32)MT_MAXM) {
    if (t == 0) atomicOr(&TG.flags, (u32)PCS_FLAG_CAPACITY);
    return;
  }
  // dummy (x, y, I0) of occupied cell b (computed where needed: the cell
  // arrays stay small enough for two CTAs per SM)
  auto dummy3 = [&](int b, float& x, float& y, float& i0) {
    const int o = sm.u.b.occ[b];
    u32 cnt;
    i128 S[3];
    i64 ix, iy;
    if (o >= 0) {
      cnt = sm.acc_cnt[s1_swz(o)];
      ix = sx0 + o % snx;
      iy = sy0 + o / snx;
      S[0] = mt_digits(sm.dig, 0, o) + (i128)cnt * f32_to_fixed(sm.ref[o % snxi], FX_STATE);
      S[1] = mt_digits(sm.dig, 1, o) + (i128)cnt * f32_to_fixed(refy[o / snxi], FX_STATE);
      S[2] = mt_digits(sm.dig, 4, o);
    } else {
      const MtHash& h = HT[-o - 1];
      cnt = h.cnt;
      ix = (i64)(h.key - 1u) % g.ncols;
      iy = (i64)(h.key - 1u) / g.ncols;
      S[0] = mt_hash_sum(h, 0);
      S[1] = mt_hash_sum(h, 1);
      S[2] = mt_hash_sum(h, 4);
    }
    float d[3];
#pragma unroll
    for (int c = 0; c < 3; ++c)
      d[c] = __double2float_rn(scalbn(__ddiv_rn(i128_to_f64_rn(S[c]), (double)cnt), -FX_STATE));
    if (P.placement == 1) {
      d[0] = __double2float_rn(__dadd_rn(g.ox, __dmul_rn((double)ix + 0.5, g.lx)));
      d[1] = __double2float_rn(__dadd_rn(g.oy, __dmul_rn((double)iy + 0.5, g.ly)));
    }
    x = d[0];
    y = d[1];
    i0 = d[2];
  };
  int bx0 = INT_MAX, bx1 = INT_MIN, by0 = INT_MAX, by1 = INT_MIN;
  for (int b = t; b < M; b += MT_THREADS) {
    float x, y, i0;
    dummy3(b, x, y, i0);
    if (x == x && y == y) {
      int xlo, xhi, ylo, yhi;
      window_of(x, y, P.spot, P.H, P.W, xlo, xhi, ylo, yhi);
      bx0 = min(bx0, xlo); bx1 = max(bx1, xhi); by0 = min(by0, ylo); by1 = max(by1, yhi);
    }
  }
  atomicMin(&sm.box[0], bx0); atomicMax(&sm.box[1], bx1);
  atomicMin(&sm.box[2], by0); atomicMax(&sm.box[3], by1);
  __syncthreads();
  PixView pv = frame_view(P.frame, P.H, P.W);
  {
    int x0 = sm.box[0], y0 = sm.box[2];
    i64 wx = (i64)sm.box[1] - x0 + 1, wy = (i64)sm.box[3] - y0 + 1;
    if (sm.box[1] >= sm.box[0] && wx * wy <= MT_STAGE) {
      for (int p = t; p < (int)(wx * wy); p += MT_THREADS)
        sm.u.b.dpix[p] = __ldg(P.frame + (i64)(y0 + p / (int)wx) * P.W + (x0 + p % (int)wx));
      pv.base = sm.u.b.dpix;
      pv.pitch = wx;
      pv.x0 = x0;
      pv.y0 = y0;
    }
  }
  __syncthreads();
  // likelihood once per occupied cell: one warp per cell (lane = window row;
  // the canonical per-thread order, pcs_lik.cuh loglik_warp) — no
  // register-resident window, so the kernel fits 64 registers without spills
  long long lmax = LLONG_MIN;
  {
    const int lane = t & 31;
    const bool f64 = P.spot.model != 0 && P.spot.f64;
    for (int b = t >> 5; b < M; b += MT_WARPS) {
      float x, y, i0;
      dummy3(b, x, y, i0);
      const double ll = f64 ? loglik_poisson64_warp(pv, x, y, i0, P.spot, lane)
                            : loglik_warp(pv, x, y, i0, P.spot, lane);
      if (lane == 0) {
        sm.u.b.ll[b] = ll;
        lmax = max(lmax, (long long)f64_to_ordered(ll));
      }
    }
  }
  atomicMax(&sm.lmax, lmax);
  __syncthreads();
  i128 e[6] = {0, 0, 0, 0, 0, 0};
  double m;
  if (!prior) {
    m = ordered_to_f64((i64)sm.lmax);
    i128 acc1[1] = {0};
    for (int b = t; b < M; b += MT_THREADS) {
      int o = sm.u.b.occ[b];
      u32 cnt = (o >= 0) ? sm.acc_cnt[s1_swz(o)] : HT[-o - 1].cnt;
      acc1[0] += (i128)cnt * f64_to_fixed(exp(__dsub_rn(sm.u.b.ll[b], m)), FX_S);
    }
    block_sum_i128_k<MT_THREADS, 1>(acc1, sm.red);
    if (t == 0) sm.Sf = scalbn(i128_to_f64_rn(acc1[0]), -FX_S);
    __syncthreads();
    const double Sf = sm.Sf;
    for (int b = t; b < M; b += MT_THREADS) {
      int o = sm.u.b.occ[b];
      float w = normalised_weight(sm.u.b.ll[b], m, Sf);
      atomicMin(&sm.wmin, __float_as_uint(w));
      atomicMax(&sm.wmax, __float_as_uint(w));
      i128 wq = f32_to_fixed(w, FX_WQ);
      u32 cnt;
      if (o >= 0) {
        sm.wfix_sub[o] = cdf_fixed(w);
        sm.wsub_f[o] = w;
        cnt = sm.acc_cnt[s1_swz(o)];
#pragma unroll
        for (int c = 0; c < 5; ++c) {
          i128 S = mt_digits(sm.dig, c, o);
          if (c == 0) S += (i128)cnt * f32_to_fixed(sm.ref[o % snxi], FX_STATE);
          if (c == 1) S += (i128)cnt * f32_to_fixed(refy[o / snxi], FX_STATE);
          e[c] += wq * S;
        }
      } else {
        MtHash& h = HT[-o - 1];
        cnt = h.cnt;
        // the sums are consumed: zero them for the next frame; the cell's
        // weight waits for phase C in sum[4][1] (cleared there)
#pragma unroll
        for (int c = 0; c < 5; ++c) e[c] += wq * mt_hash_sum(h, c);
        mt_hash_clear(h);
        h.stash = (u64)__float_as_uint(w);
      }
      e[5] += (i128)cnt * f64_to_fixed((double)w * (double)w, FX_W2);
    }
  } else {
    // prior weights: the cell log-likelihoods by cell code (sub-window table
    // aliasing wfix_sub; outlier cells in their hash slot, sums zeroed)
    double* llsub = reinterpret_cast<double*>(sm.wfix_sub);
    for (int b = t; b < M; b += MT_THREADS) {
      const int o = sm.u.b.occ[b];
      const double llb = sm.u.b.ll[b];
      if (o >= 0) {
        llsub[o] = llb;
      } else {
        MtHash& h = HT[-o - 1];
        mt_hash_clear(h);
        h.stash = (u64)__double_as_longlong(llb);
      }
    }
    __syncthreads();
    // log w = log w_prev + ll[cell] and its maximum (k_pc_prior_ll)
    long long pm = LLONG_MIN;
    bool nf = false;
    for (i64 j = t; j < n; j += MT_THREADS) {
      const u32 code = P.pslot[base_i + j];
      const double llc = (code & 0x80000000u)
                             ? __longlong_as_double((long long)HT[mt_hash_find(HT, code & 0x7FFFFFFFu)].stash)
                             : llsub[code];
      const double ll = __dadd_rn(log((double)P.wprev[base_i + j]), llc);
      P.ll[base_i + j] = ll;
      if (!(ll == ll) || ll == INFINITY) nf = true;
      pm = max(pm, (long long)f64_to_ordered(ll));
    }
    if (nf) atomicOr(&TG.flags, (u32)PCS_FLAG_NONFINITE);
    atomicMax(&sm.plmax, pm);
    __syncthreads();
    m = ordered_to_f64((i64)sm.plmax);
    // S = sum round(exp(log w - m) 2^95), exp(log w - m) kept per particle (k_sir_sum)
    i128 acc1[1] = {0};
    for (i64 j = t; j < n; j += MT_THREADS) {
      const double ex = exp(__dsub_rn(P.ll[base_i + j], m));
      P.ll[base_i + j] = ex;
      acc1[0] += f64_to_fixed(ex, FX_S);
    }
    block_sum_i128_k<MT_THREADS, 1>(acc1, sm.red);
    if (t == 0) sm.Sf = scalbn(i128_to_f64_rn(acc1[0]), -FX_S);
    __syncthreads();
    const double Sf = sm.Sf;
    // estimate / ESS numerators per particle (k_sir_stats)
    unsigned wmn = 0xFFFFFFFFu, wmx = 0u;
    for (i64 j = t; j < n; j += MT_THREADS) {
      const float w = weight_from_ex(P.ll[base_i + j], Sf);
      wmn = min(wmn, __float_as_uint(w));
      wmx = max(wmx, __float_as_uint(w));
      const i128 wq = f32_to_fixed(w, FX_WQ);
#pragma unroll
      for (int c = 0; c < 5; ++c) e[c] += wq * f32_to_fixed(sout[c * ld + base_i + j], FX_STATE);
      e[5] += f64_to_fixed((double)w * (double)w, FX_W2);
    }
    atomicMin(&sm.wmin, wmn);
    atomicMax(&sm.wmax, wmx);
  }
  const bool bad_m = !(m == m) || m == INFINITY;
  const bool degenerate = (m == -INFINITY);
  block_sum_i128_k<MT_THREADS, 6>(e, sm.red);
  __shared__ int s_res, s_keep;
  if (t == 0) {
    const i64 row = tg * P.K + k;
    double ess = 1.0 / scalbn(i128_to_f64_rn(e[5]), -FX_W2);
    bool flag_bad = degenerate || bad_m;
    if (degenerate) atomicOr(&TG.flags, (u32)PCS_FLAG_DEGENERATE);
    if (bad_m) atomicOr(&TG.flags, (u32)PCS_FLAG_NONFINITE);
    if (flag_bad) atomicMin(&TG.first_bad, (int)k);
    double est[5];
    for (int c = 0; c < 5; ++c) {
      est[c] = scalbn(i128_to_f64_rn(e[c]), -(FX_WQ + FX_STATE));
      P.out_est[row * 5 + c] = est[c];
    }
    P.out_ess[row] = ess;
    int res = (!flag_bad && ess < P.thresh) ? 1 : 0;   // filtering.py:169-170
    // without resampling the next frame starts from these weights unless they
    // are all equal (then uniform, as the single-target loop does)
    int keep = (!res && !flag_bad && sm.wmin != sm.wmax) ? 1 : 0;
    if (keep && !P.wprev) {   // (threshold 1: ESS rounded up to n with unequal weights)
      atomicOr(&TG.flags, (u32)PCS_FLAG_CAPACITY);
      keep = 0;
    }
    TG.prior = keep;
    TG.span = (sm.obox[0] <= sm.obox[1])
                  ? max(sm.obox[1] - sm.obox[0], sm.obox[3] - sm.obox[2]) + 1 : 0;
    s_keep = keep;
    P.out_res[row] = (unsigned char)res;
    P.out_occ[row] = M;
    TG.evals += M;
    if (!flag_bad) {
      TG.center[0] = est[0];
      TG.center[1] = est[1];
    }
    s_res = res;
    sm.carry = 0;
  }
  __syncthreads();

  // ---------------- phase C: exact-prefix resampling ----------------
  // (k_sys_resample in one CTA: scan tiles of 2560 particles in order, exact
  // u128 prefixes, first slot per item from the top 64 bits of the prefix,
  // run heads + block max-scan, coalesced ancestor writes; multinomial: the
  // exact cdf per particle, then k_multinomial_emit's search)
  const int do_res = s_res, keep = GEN && s_keep;
  const bool multi = GEN && P.multinomial != 0;
  const double Sfr = sm.Sf;
  const double u = philox_resample_u(seed_t, P.frame0 + (u32)k);
  constexpr int CI = MT_CI;
  constexpr int CT = MT_CT;
  u32* cells = sm.u.c.cells;
  int* hp = reinterpret_cast<int*>(sm.u.c.cells);   // item k's run head over its cell
  int* stage = sm.u.c.stage;
  const double nd = (double)n, eps = nd * 8.881784197001252e-16;   // n * 2^-50
  const double kappa = nd * 1.0842021724855044e-19;                  // n * 2^-63
  // exact weight of a staged particle: sub-window cell table, else the hash
  auto cellw = [&](u32 code) -> u128 {
    if (code == 0xFFFFFFFFu) return 0;
    if (!(code & 0x80000000u)) return sm.wfix_sub[code];
    const u32 key = (code & 0x7FFFFFFFu) + 1u;
    u32 s = mt_hash_slot(key);
    for (int probe = 0; probe < MT_HCAP; ++probe) {
      if (HT[s].key == key) return cdf_fixed(__uint_as_float((u32)HT[s].stash));
      s = (s + 1u) & (MT_HCAP - 1);
    }
    return 0;
  };
  // exact weight of item kk of the scan tile at `base` (prior frames: per particle)
  auto itemw = [&](int kk, i64 base, int nv) -> u128 {
    if (!prior) return cellw(cells[kk]);
    return (kk < nv) ? cdf_fixed(weight_from_ex(P.ll[base_i + base + kk], Sfr)) : (u128)0;
  };
  u128 pre = 0;
  i64 tj_prev = 0;
  const int k0 = t * CI;
  for (i64 base = 0; base < n; base += CT) {
    if (!do_res) {
      for (int q = 0; q < CI; ++q) {
        const i64 i = base + (i64)q * MT_THREADS + t;
        if (i < n) {
          P.anc[base_i + i] = (int)i;
          if (keep) {   // the particles keep their weights (filtering.py:171)
            float w;
            if (prior) {
              w = weight_from_ex(P.ll[base_i + i], Sfr);
            } else {
              const u32 code = P.pslot[base_i + i];
              w = (code & 0x80000000u)
                      ? __uint_as_float((u32)HT[mt_hash_find(HT, code & 0x7FFFFFFFu)].stash)
                      : sm.wsub_f[code];
            }
            P.wprev[base_i + i] = w;
          }
        }
      }
      continue;
    }
    const int nv = (int)min((i64)CT, n - base);   // items of this scan tile
    for (int q = 0; q < CI; ++q) {
      const int idx = q * MT_THREADS + t;
      cells[idx] = (idx < nv) ? P.pslot[base_i + base + idx] : 0xFFFFFFFFu;
    }
    __syncthreads();
    u128 tsum = 0;
#pragma unroll
    for (int q = 0; q < CI; ++q) tsum += itemw(k0 + q, base, nv);
    u128 inc = tsum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      u128 o = shfl_up_u128(inc, d);
      if (lane >= d) inc += o;
    }
    if (lane == 31) sm.wtot[warp] = inc;
    __syncthreads();
    u128 woff, tagg;
    {   // every warp scans the MT_WARPS warp totals with shuffles (no extra barrier)
      const u128 wv = (lane < MT_WARPS) ? sm.wtot[lane] : (u128)0;
      u128 wi = wv;
#pragma unroll
      for (int d = 1; d < MT_WARPS; d <<= 1) {
        const u128 o = shfl_up_u128(wi, d);
        if (lane >= d) wi += o;
      }
      woff = shfl_u128(wi - wv, warp);
      tagg = shfl_u128(wi, MT_WARPS - 1);
    }
    const u128 excl = pre + woff + (inc - tsum);
    const bool last_tile = base + CT >= n;
    const int klast = last_tile ? nv - 1 : -1;   // the target's last particle ends at slot n
    if (multi) {   // the exact cdf (filtering.py:94-95); the search follows the scan
      u128 run = excl;
#pragma unroll
      for (int q = 0; q < CI; ++q) {
        const int kk = k0 + q;
        if (kk < nv) {
          run += itemw(kk, base, nv);
          P.cdf[base_i + base + kk] = (kk == klast) ? 1.0 : cdf_round(run);
        }
      }
      pre += tagg;
      __syncthreads();   // (wtot is rewritten by the next tile)
      continue;
    }
    const i64 tj0 = tj_prev;   // a tile starts where the previous one ended
    const i64 tj1 = last_tile ? n : first_slot_fast(cdf_round(pre + tagg), u, n, nd, eps);
    tj_prev = tj1;
    {
      const double tj0d = (double)tj0;
      int jr = 0;
      if (k0 < nv && base + k0 != 0) jr = slot_rel(excl, u, n, nd, kappa, eps, tj0d, tj0);
      u128 run = excl;
#pragma unroll
      for (int q = 0; q < CI; ++q) {
        const int kk = k0 + q;
        int h = -1;   // no slot
        if (kk < nv) {
          run += itemw(kk, base, nv);
          const int jend = (kk == klast) ? (int)(n - tj0) : slot_rel(run, u, n, nd, kappa, eps, tj0d, tj0);
          if (jend > jr) h = jr;
          jr = jend;
        }
        hp[kk] = h;
      }
    }
    __syncthreads();
    const int m_slots = (int)(tj1 - tj0);   // <= n < 2^31
    int carry = -1;
    for (int c0 = 0; c0 < m_slots; c0 += CT) {
#pragma unroll
      for (int q = 0; q < CI; ++q) stage[k0 + q] = -1;
      __syncthreads();
#pragma unroll
      for (int q = 0; q < CI; ++q) {
        const u32 hr = (u32)(hp[k0 + q] - c0);   // no head: (u32)(-1 - c0) >= 2^31
        if (hr < (u32)CT) stage[hr] = k0 + q;
      }
      __syncthreads();
      int tmax = -1;
#pragma unroll
      for (int q = 0; q < CI; ++q) tmax = max(tmax, stage[k0 + q]);
      int incl = tmax;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl = max(incl, o);
      }
      if (lane == 31) sm.scan_tmp[warp] = incl;
      int excl_l = __shfl_up_sync(0xffffffffu, incl, 1);
      if (lane == 0) excl_l = -1;
      __syncthreads();
      int prev = carry, total = carry;
      for (int w = 0; w < MT_WARPS; ++w) {
        if (w < warp) prev = max(prev, sm.scan_tmp[w]);
        total = max(total, sm.scan_tmp[w]);
      }
      int runm = max(prev, excl_l);
#pragma unroll
      for (int q = 0; q < CI; ++q) {
        runm = max(runm, stage[k0 + q]);
        stage[k0 + q] = runm;
      }
      __syncthreads();
      const int cm = min(CT, m_slots - c0);
      int* out = P.anc + base_i + tj0 + c0;
      const int ib = (int)base;
      for (int kk = t; kk < cm; kk += MT_THREADS) __stcs(out + kk, ib + stage[kk]);   // (evict-first)
      carry = total;
      __syncthreads();
    }
    pre += tagg;
  }
  if (do_res && multi) {
    // ancestor j = searchsorted(cdf, p_j, 'right') over the target's exact cdf,
    // p_j = philox_multinomial_u(seed_t, frame, j) (filtering.py:96-97,100)
    __syncthreads();   // the cdf writes of every thread are visible
    const double* cdf = P.cdf + base_i;
    const u32 f = P.frame0 + (u32)k;
    for (i64 j = t; j < n; j += MT_THREADS) {
      const double p = philox_multinomial_u(seed_t, f, (u64)j);
      i64 lo = 0, hi = n;   // first index with cdf > p
      while (lo < hi) {
        const i64 mid = (lo + hi) >> 1;
        if (cdf[mid] <= p) lo = mid + 1;
        else hi = mid;
      }
      P.anc[base_i + j] = (int)((lo < n) ? lo : n - 1);
    }
  }
  // clear the consumed outlier cells for the next frame (after every thread's
  // last read of them: the identity path above reads weights without a barrier)
  __syncthreads();
  for (int s = t; s < MT_HCAP; s += MT_THREADS) {
    if (HT[s].key) {
      HT[s].key = 0u;
      HT[s].cnt = 0u;
      HT[s].stash = 0ull;
    }
  }
}

constexpr size_t MT_SMEM = sizeof(MtSmem);

}  // namespace pcs
