// pcs_fused.cuh — fused per-frame kernels of the device-resident filter loop.
//
//   k_pc_step1      gather (resampling, filtering.py:107) + propagate
//                   (state.py:115-127) + cell index (binning.py:61-67,105) +
//                   exact per-cell sums for the dummies (binning.py:157-172)
//                   in ONE pass over the particle states.
//   k_pc_cells / k_pc_bins   per-cell dummies + likelihoods, then the
//                   normaliser / weights / estimate / ESS / decision
//   k_sys_resample  exact-prefix systematic resampling (filtering.py:93-100)
//
// Per-cell accumulation without 64-bit shared-memory atomics (those are CAS
// loops on sm_100): 32-bit digit accumulators (S1Smem).
// Integer sums are order-free, so the result is exactly the canonical sum of
// round(s * 2^40).
#pragma once
#include "pcs_common.cuh"
#include "pcs_lik.cuh"
#include "pcs_state.cuh"
#include "pcs_weights.cuh"

namespace pcs {

#ifndef PCS_S1_THREADS
#define PCS_S1_THREADS 256
#endif
#ifndef PCS_S1_DEEP
#define PCS_S1_DEEP 1   // k_pc_step1: the next chunk's states in registers too
#endif
constexpr int S1_THREADS = PCS_S1_THREADS;     // 2 CTAs x 16 warps per SM; 64 registers
#ifndef PCS_S1_CTAS
#define PCS_S1_CTAS 2
#endif
#ifndef PCS_S1_IPT
#define PCS_S1_IPT 3
#endif
constexpr int S1_CTAS_PER_SM = PCS_S1_CTAS;
constexpr int S1_IPT = PCS_S1_IPT;             // particles per lane per chunk
constexpr int S1_WARPS = S1_THREADS / 32;
constexpr int S1_SIDE = 32;                    // sub-window side (cells)
constexpr int SUBW = S1_SIDE * S1_SIDE;        // shared-memory sub-window cells
constexpr int S1_PARTS = 15;                   // 5 components x 3 digits (16/16/signed)
constexpr int S1_MAX_WT = 2048;                // most particles per warp tile
// a sub-window cell's digits are flushed (taken by atomic exchange) each
// time its count crosses a multiple of S1_CELL_FLUSH, so between two flushes
// a digit gets S1_CELL_FLUSH additions plus those in flight (< 2 per resident
// thread): < 2^16 additions of < 2^16 (|.| <= 2^15 for the signed digit), no
// 32-bit accumulator wraps
constexpr u32 S1_CELL_FLUSH = 16384;
constexpr i64 TABLE_MAX = 0xFFFFFFFFll;        // grid cells (flat ids are u32; 2^32 - 1 = empty key)
// per-frame cell table: open addressing over HT_CAP slots keyed by the flat
// cell id (2x the occupied-cell capacity MAXM), instead of a dense full-grid
// table (28 GB at config 5's 16384^2 grid)
constexpr int HT_BITS = 21;
constexpr u32 HT_CAP = 1u << HT_BITS;
constexpr u32 HT_EMPTY = 0xFFFFFFFFu;
constexpr int MAXM = 1 << 20;                  // occupied cells per frame (fused)

// k_pc_step1 (two 256-thread CTAs per SM, 3 particles per lane per chunk, the
// next chunk's ancestors and states loaded while the current one computes):
// every warp runs its own tiles of particles — gather, propagate, cell — and
// adds each particle that lands in the frame's 32x32-cell shared-memory
// sub-window (cells at bank-swizzled slots, s1_swz) to
// that cell's exact fixed-point sums with native 32-bit shared atomics: the
// int64 value V = round(v 2^40) of each component goes into three 32-bit
// digit accumulators (bits 0-15, 16-31, V >> 32). There are no CTA barriers
// inside the particle loop. Integer sums are order-free, so the cell sums are
// exactly the canonical sums of round(s 2^40); the CTA folds
// them into the int128 HBM table at the end (s1_flush) and a cell whose count
// crosses a multiple of S1_CELL_FLUSH is folded on the spot (s1_cell_flush).
// Particles outside the sub-window add to the table directly (limb
// reductions) — on the spot in the steady-state instantiation, from a
// per-warp queue, 32 per batch, in the one the first frame of a track runs
// (QUEUE; the initial cloud is usually wider than the sub-window).
constexpr int S1_CHUNK = 32 * S1_IPT;          // particles per warp pipeline step
constexpr int S1_OQ = 32 + S1_CHUNK;           // queue entries per warp (< 32 left + one chunk)
struct S1Smem {
  u32 dig[S1_PARTS][SUBW];
  u32 cnt[SUBW];          // in-window members of each cell (this CTA)
  float ref[SUBW + 1];    // cell lower edges: x at [0, snx), y at [snx, snx + sny)
                          // (NaN: deltas from this edge may not be exact)
  int fast_delta;
  // table pointers for the out-of-line cell flush (read only on that path)
  u32* fl_hkey;
  int fl_shift;
  u64* fl_tab_sum;
  u32* fl_occ;
  i64 fl_G;
};

// k_pc_step1<., true> only (behind S1Smem in its dynamic shared memory): per-warp
// queue of particles outside the sub-window (cell; particle index, bit 31:
// its cell code is already written) and its length
struct S1Queue {
  u32 oq[S1_WARPS][S1_OQ][2];
  u32 oqn[S1_WARPS];
};

struct TrackCtl {
  // ---- per frame (reset at the end of the frame for the next one)
  i64 max_ll_ord;            // SIR: ordered-int64 max loglik (float64)
  u32 n_occ;                 // pcSIR: first-touch occupied list length
  u32 wmin_bits, wmax_bits;  // SIR: min/max normalised weight (non-negative float bits)
  u32 pad_a;
  u64 S[2];                  // SIR: normaliser
  u64 est[5][2];             // SIR: estimate numerators
  u64 w2[2];                 // SIR: ESS denominator
  // ---- sub-window of the current frame
  i64 sx0, sy0, snx, sny;
  // ---- scalars consumed by the scan / emission kernel
  double m, Sf, u;
  int do_resample;
  int pad1;
  // ---- persistent
  i64 k;                     // absolute frame index (since begin)
  i64 k_frames;              // frame index of frames[0]
  i64 k_out;                 // frame index of out[0]
  const float* frames;
  double* out_est;
  double* out_ess;
  unsigned char* out_res;
  i64* out_occ;
  u32 flags;
  int first_bad;
  i64 evals;
  double center[2];          // previous estimate (shared-memory sub-window centre)
  long long dbg[16];         // phase timestamps (globaltimer ns) of the bins kernel
  unsigned long long tile_ctr;  // decoupled look-back: monotone tile ticket counter
  u64 rank_prefix[2];        // sharded: exact cumulative weight of the preceding ranks
  i64 shard_lo, shard_hi;    // sharded: this rank's emitted global slots [lo, hi)
  i64 shard_send[2];         // sharded: slots sent to rank r-1 / r+1 this frame
  i64 shard_recv[2];         // sharded: slots received from rank r-1 / r+1
  u32 gbar_cnt, gbar_gen;    // grid barrier of k_sys_resample
  u32 stats_done;            // k_sir_stats CTAs finished (the last one finalises)
  u32 s1_ticket, s1_done;    // k_pc_step1 dynamic tile tickets (reset by its last CTA)
  u32 sir_ticket, sir_done;  // k_sir_propagate_lik dynamic chunk tickets
  u32 res_frame;             // RNG frame of this frame's resampling (multinomial points)
  int fmap_ok;               // P.fmap describes the current frame batch (TMA staging)
  int prior_nonuniform;      // the NEXT frame starts from the prior weights wprev (no
                             // resampling at this frame, weights not all equal)
  int pc_prior;              // pcSIR: THIS frame has prior weights (copied from
                             // prior_nonuniform by k_pc_step1 at the frame start)
  i64 frame_occ;             // pcSIR with prior weights: occupied cells of the frame
  i64 k_end;                 // frame index one past the last output row of this batch
  i64 cell_max_ord;          // pcSIR: ordered-int64 max cell log-likelihood (k_pc_cells)
  u32 s1_mid_flush;          // diagnostics: step-1 per-cell exchange flushes (pcs_track_info)
  u32 max_occ;               // diagnostics: most occupied cells of a frame
};

// cell-index constants of one grid axis (cell_axis_hot below)
struct AxisFast {
  float o32, inv32, mt, ma, mb, fmax;
  u32 imax;              // (u32)fmax
  double origin, cell, inv;
  i64 n;
};

struct TrackParams {
  i64 n, ld;
  i64 H, W;
  Dyn dyn;
  Spot spot;
  Grid grid;
  double inv_lx, inv_ly;
  AxisFast axx, axy;         // k_pc_step1 cell index constants (make_axis on the host)
  u64 seed;
  PhiloxKey pk;              // round keys of seed (constant-bank operands)
  u32 frame0;
  int placement;
  int weighted;              // pcSIR weighted centre of mass (uniform prior weights only)
  float* buf0;
  float* buf1;
  int* anc;
  double* ll;                // SIR: per-particle log-likelihood (float64); k_sir_sum
                             // replaces it by exp(ll - max) for the rest of the frame
  u32* pslot;                // pcSIR: cell code per particle (pslot_code below)
  u32* hkey;                 // [G] flat cell id of each table slot (HT_EMPTY: free)
  int ht_shift;              // log2(columns) when that is a power of two (bit-slice hash), else -1
  u32* tab_cnt;              // [G]   members per slot
  u64* tab_sum;              // [5][G][2] exact int128 sums (step-1 flushes, shard import)
  u64* tab_lim;              // [5][G][3] limb sums (step-1 single particles, tab_add)
  float* wtab;               // [G]
  u128* wfix;                // [G] exact cdf weight round(wtab * 2^120) (k_sys_resample)
  u32* occ;                  // [MAXM]
  i64 G;                     // table slots (HT_CAP)
  i64 ntiles;                // scan tiles
  u32* tile_status;          // [ntiles] (frame tag << 2 | state)
  u128* tile_agg;            // [ntiles]
  u128* tile_inc;            // [ntiles]
  TrackCtl* ctl;
  // ---- particle sharding (config 5); single GPU: 0, n, 0, n, anc
  i64 idx_off;               // global index of local particle 0 (Philox counter)
  i64 n_global;              // particles over all ranks
  i64 slot_lo;               // first global output slot emitted by this rank
  i64 slot_cap;              // capacity of anc_out
  int* anc_out;              // ancestors (local particle index) for slots slot_lo + k
  int scan_mode;             // k_sys_resample: 0 both passes, 1 pass 1 only, 2 pass 2 only
  int sharded;               // particle-sharded filter: a frame with prior weights is
                             // finalised after the all-reduce of its per-particle sums
                             // (k_shard_prior_in), not by k_sir_stats
                             // (sharded: rank prefix and first slot in ctl)
  int s1_tile;               // k_pc_step1 warp tile (<= S1_MAX_WT), balanced over the warps
  double thresh;             // resample when ESS < thresh (= threshold_fraction * N)
  float* wprev;              // normalised prior weights when prior_nonuniform
  double* lltab;             // pcSIR with prior weights: [G] log-likelihood per cell
  u128* wsub;                // [SUBW] wfix of the frame's step-1 sub-window cells (by code); == wfix - SUBW
  double* ltsub;             // [SUBW] lltab of the sub-window cells
  float* wtsub;              // [SUBW] wtab of the sub-window cells
  int method;                // 0 SIR, 1 pcSIR
  int sir_chunk;             // k_sir_propagate_lik: particles per dynamic chunk
  int multinomial;           // resampling scheme: the resampler writes the cdf and
  double* cdf;               // [N] k_multinomial_emit searches it
  const void* fmap;          // device CUtensorMap of the frame batch [K][H][W] f32,
                             // boxes of FMAP_BX x FMAP_BY pixels (TMA staging)
  u128* cta_agg;             // k_sys_resample: per-CTA exact weight totals
};

// pcSIR cell code of a particle (P.pslot): the cell's index q < SUBW in the
// frame's step-1 sub-window (row-major, snx columns), else SUBW + its flat id.
// Per-cell tables are read through the code: the sub-window cells from the
// compact per-frame tables (16 KB for wsub, L1-resident), the others from the
// full-grid tables.
__device__ __forceinline__ u128 code_wfix(const TrackParams& P, u32 code) {
  return P.wsub[code];   // wfix == wsub + SUBW (pcs_track_begin): one 16-byte load, no select
}
__device__ __forceinline__ float code_wtab(const TrackParams& P, u32 code) {
  return code < (u32)SUBW ? P.wtsub[code] : P.wtab[code - SUBW];
}
__device__ __forceinline__ double code_ll(const TrackParams& P, u32 code) {
  return code < (u32)SUBW ? P.ltsub[code] : P.lltab[code - SUBW];
}
// the sub-window code of flat cell id `cell` (bins kernel), or -1
__device__ __forceinline__ int sub_code(const TrackParams& P, const TrackCtl* C, u32 cell) {
  const u32 nc = (u32)P.grid.ncols;
  const u32 iy = cell / nc, ix = cell - iy * nc;
  const i64 qx = (i64)ix - C->sx0, qy = (i64)iy - C->sy0;
  if (qx < 0 || qx >= C->snx || qy < 0 || qy >= C->sny) return -1;
  return (int)(qy * C->snx + qx);
}

// Programmatic dependent launch: the frame's kernels are launched with the
// programmatic-serialization attribute, so the next kernel is scheduled while
// the current one drains; it waits here for the previous grid (complete and
// visible) before touching its results.
__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ void set_flag(TrackCtl* c, u32 f) {
  atomicOr(&c->flags, f);
  atomicMin(&c->first_bad, (int)c->k);
}

__device__ __forceinline__ void reset_frame(TrackCtl* c) {
  c->max_ll_ord = LLONG_MIN;
  c->cell_max_ord = LLONG_MIN;
  c->n_occ = 0;
  c->wmin_bits = 0xFFFFFFFFu;
  c->wmax_bits = 0u;
  c->S[0] = c->S[1] = 0;
  for (int q = 0; q < 5; ++q) c->est[q][0] = c->est[q][1] = 0;
  c->w2[0] = c->w2[1] = 0;
}

// ---------------------------------------------------------------------------
// fast exact cell index: floor(RN((p - o)/l)) without a division unless the
// multiplied quotient is within a few ulps of an integer (CANONICAL result is
// identical to cell_axis in pcs_common.cuh)
// ---------------------------------------------------------------------------
__device__ __forceinline__ i64 cell_axis_fast(float p, double origin, double cell, double inv,
                                              i64 n) {
  // float32 estimate first: accepted when its fractional part is farther from
  // an integer than its error bound (|p|+|o|)|1/l| 2^-20 + |t| 2^-20
  {
    float o32 = (float)origin, inv32 = (float)inv;
    float t32 = (p - o32) * inv32;
    float f32 = floorf(t32);
    float fr32 = t32 - f32;
    float margin = ((fabsf(p) + fabsf(o32)) * fabsf(inv32) + fabsf(t32) + 1.0f) *
                   9.5367431640625e-07f;
    if (fr32 > margin && fr32 < 1.0f - margin) {
      if (!(f32 >= 0.0f)) return 0;
      if ((double)f32 > (double)(n - 1)) return n - 1;
      return (i64)f32;
    }
  }
  double d = __dsub_rn((double)p, origin);
  double t = __dmul_rn(d, inv);
  double f = floor(t);
  double fr = t - f;
  double margin = fabs(t) * 3.552713678800501e-15 + 1e-300;  // |t| * 2^-48
  double q = (fr > margin && fr < 1.0 - margin) ? f : floor(__ddiv_rn(d, cell));
  if (!(q >= 0.0)) return 0;
  double hi = (double)(n - 1);
  if (q > hi) return n - 1;
  return (i64)q;
}

// Hot-loop form of cell_axis_fast with the per-axis constants hoisted. The
// float32 estimate t32 = (p - o32) * inv32 is accepted when its fractional
// part is farther from an integer than the margin
//   general:            ((|p| + |o32|)|inv32| + |t32| + 1) 2^-20 (cell_axis_fast)
//   pow2 cell, o32 = o: 0, i.e. t32 not an integer
// (with a power-of-two cell and a float32-exact origin the product is exact
// and the only error is the round-to-nearest of p - o32; rounding is
// monotone and the cell edges o + k l are float32 values, so the rounded
// quotient has the exact quotient's floor unless it lands exactly ON an
// integer), and only inside [0, min(n-1, 2^24)]; everything else (integer
// quotients, clamping, NaN) takes the float64 path. Same result as
// cell_axis_fast.

__host__ __device__ __forceinline__ AxisFast make_axis(double origin, double cell, double inv, i64 n) {
  AxisFast a;
  a.o32 = (float)origin;
  a.inv32 = (float)inv;
  int e;
#ifdef __CUDA_ARCH__
  const double ci = __dmul_rn(cell, inv);
#else
  const double ci = cell * inv;
#endif
  const bool pow2 = frexp(inv, &e) == 0.5 && ci == 1.0 &&
                    (double)a.inv32 == inv && (double)a.o32 == origin && e > -100 && e < 100;
  if (pow2) {
    a.mt = 0.0f;
    a.ma = 0.0f;
    a.mb = 0.0f;
  } else {
    a.mt = 9.5367431640625e-07f;     // 2^-20
    a.ma = fabsf(a.inv32) * 9.5367431640625e-07f;
    a.mb = (fabsf(a.o32) * fabsf(a.inv32) + 1.0f) * 9.5367431640625e-07f;
  }
  a.fmax = (float)(n - 1 < (i64)(1 << 24) ? n - 1 : (i64)(1 << 24));
  a.imax = (u32)(n - 1 < (i64)(1 << 24) ? n - 1 : (i64)(1 << 24));
  a.origin = origin;
  a.cell = cell;
  a.inv = inv;
  a.n = n;
  return a;
}

// POW2: both axes have power-of-two cells and float32-exact origins (the
// margins are zero, see make_axis): only an integer quotient is ambiguous
template <bool POW2>
__device__ __forceinline__ int cell_axis_hot(float p, const AxisFast& a) {
  const float t32 = __fmul_rn(__fsub_rn(p, a.o32), a.inv32);
  const float f32 = floorf(t32);
  const float fr32 = t32 - f32;
  if (POW2) {
    // (floor as an integer; an integer quotient or a value outside [0, fmax]
    // takes the float64 path)
    const int i = __float2int_rd(t32);
    if ((float)i != t32 && (u32)i <= a.imax) return i;
  } else {
    const float margin = fmaf(fabsf(t32), a.mt, fmaf(fabsf(p), a.ma, a.mb));
    if (fr32 > margin && fr32 < 1.0f - margin && f32 >= 0.0f && f32 <= a.fmax)
      return __float2int_rz(f32);
  }
  return (int)cell_axis_fast(p, a.origin, a.cell, a.inv, a.n);
}
// host: both axes of the grid take the POW2 form of cell_axis_hot
__host__ __forceinline__ bool grid_pow2(double origin_x, double lx, double origin_y, double ly) {
  auto axis = [](double o, double l) {
    const double inv = 1.0 / l;
    int e;
    return std::frexp(inv, &e) == 0.5 && l * inv == 1.0 && (double)(float)inv == inv &&
           (double)(float)o == o && e > -100 && e < 100;
  };
  return axis(origin_x, lx) && axis(origin_y, ly);
}

// cell lower edge as float32 and whether it is an integer multiple of 2^-40
__device__ __forceinline__ float cell_ref32(double origin, double cell, i64 i, bool& ok) {
  float r = __double2float_rn(__dadd_rn(origin, __dmul_rn((double)i, cell)));
  ok = (r == 0.0f) || (fabsf(r) >= 7.62939453125e-06f);  // |r| >= 2^-17 -> lsb >= 2^-40
  return r;
}


// table slot of flat cell id `flat` (inserted if absent; HT_EMPTY if the
// table is full): Fibonacci hash, linear probing; keys only go from empty to
// a cell id within a frame (the bins kernel clears the occupied slots)
// (sh >= 0: the grid has 2^sh columns — the slot is a bit slice of (row,
// column), so the cells of a cloud never collide and neighbouring cells get
// neighbouring slots: the weight lookups of the particles outside the
// sub-window, frame 0 of a track, then share sectors and lines)
__device__ __forceinline__ u32 ht_hash(u32 flat, int sh) {
  if (sh >= 0) return (((flat >> sh) & ((HT_CAP >> 11) - 1u)) << 11) | (flat & 2047u);
  return (flat * 0x9E3779B1u) >> (32 - HT_BITS);
}
__device__ __forceinline__ u32 ht_insert(const TrackParams& P, u32 flat, bool& created) {
  created = false;
  u32 s = ht_hash(flat, P.ht_shift);
  for (u32 probe = 0; probe < HT_CAP; ++probe) {
    const u32 k = __ldcg(P.hkey + s);
    if (k == flat) return s;
    if (k == HT_EMPTY) {
      const u32 old = atomicCAS(P.hkey + s, HT_EMPTY, flat);
      created = (old == HT_EMPTY);
      if (old == HT_EMPTY || old == flat) return s;
    }
    s = (s + 1) & (HT_CAP - 1);
  }
  return HT_EMPTY;
}
__device__ __forceinline__ u32 ht_insert(const TrackParams& P, u32 flat) {
  bool created;
  return ht_insert(P, flat, created);
}
__device__ __forceinline__ u32 ht_find(const TrackParams& P, u32 flat) {
  u32 s = ht_hash(flat, P.ht_shift);
  for (u32 probe = 0; probe < HT_CAP; ++probe) {
    const u32 k = __ldcg(P.hkey + s);
    if (k == flat) return s;
    if (k == HT_EMPTY) return HT_EMPTY;
    s = (s + 1) & (HT_CAP - 1);
  }
  return HT_EMPTY;
}

// add cnt members to table slot `slot`; the first touch appends the slot to
// the frame's occupied list
// A cell's exact sum of component c is tab_sum (int128, added with a carry
// chain by the step-1 flushes: few, large additions) plus tab_lim: three
// 64-bit limbs (bits 0-31 and 32-63 unsigned, the rest signed) that single
// particles outside the sub-window add with fire-and-forget reductions (RED,
// no return value), so a warp never waits on an L2 round trip per particle.
// A limb gains < 2^32 per addition and a cell gets < 2^32 additions per
// frame (n < 2^31), so none wraps.
constexpr int TAB_LIMBS = 3;
__device__ __forceinline__ u64* tab_ptr(const TrackParams& P, int c, u32 slot) {
  return P.tab_lim + ((i64)c * P.G + slot) * TAB_LIMBS;
}
__device__ __forceinline__ void tab_add(u64* p, i128 v) {
  const u128 u = (u128)v;
  const u64 l0 = (u64)u & 0xFFFFFFFFull, l1 = (u64)(u >> 32) & 0xFFFFFFFFull;
  const u64 l2 = (u64)(long long)(v >> 64);   // arithmetic shift: the signed rest
  if (l0) atomicAdd((unsigned long long*)p, l0);
  if (l1) atomicAdd((unsigned long long*)p + 1, l1);
  if (l2) atomicAdd((unsigned long long*)p + 2, l2);
}
__device__ __noinline__ void tab_add_slow(u64* p, float v) { tab_add(p, f32_to_fixed(v, FX_STATE)); }
// round(v 2^40) of one float32 state value into the limbs: for 2^-17 <= |v| <
// 2^23 (and 0) the product is an exact int64 (no rounding), else the
// general conversion
__device__ __forceinline__ void tab_add_f32(u64* p, float v) {
  const float av = fabsf(v);
  if (av < 8388608.0f && (av >= 7.62939453125e-06f || av == 0.0f)) {
    const long long x = __float2ll_rn(__fmul_rn(v, 1099511627776.0f));
    const u64 l0 = (u64)x & 0xFFFFFFFFull, l1 = ((u64)x >> 32) & 0xFFFFFFFFull;
    if (l0) atomicAdd((unsigned long long*)p, l0);
    if (l1) atomicAdd((unsigned long long*)p + 1, l1);
    if (x < 0) atomicAdd((unsigned long long*)p + 2, ~0ull);   // the signed rest: -1
  } else {
    tab_add_slow(p, v);
  }
}
__device__ __forceinline__ void tab_add_x5(const TrackParams& P, u32 slot, const i128 (&v)[5]) {
#pragma unroll
  for (int c = 0; c < 5; ++c) tab_add(tab_ptr(P, c, slot), v[c]);
}
__device__ __forceinline__ u64* tab_i128(const TrackParams& P, int c, u32 slot) {
  return P.tab_sum + ((i64)c * P.G + slot) * 2;
}
__device__ __forceinline__ i128 tab_load(const TrackParams& P, int c, u32 slot) {
  const u64* p = tab_ptr(P, c, slot);
  return load_i128(tab_i128(P, c, slot)) + (i128)p[0] + ((i128)p[1] << 32) +
         ((i128)(long long)p[2] << 64);
}
__device__ __forceinline__ void tab_zero(const TrackParams& P, int c, u32 slot) {
  u64* p = tab_ptr(P, c, slot);
  p[0] = 0;
  p[1] = 0;
  p[2] = 0;
  u64* q = tab_i128(P, c, slot);
  q[0] = 0;
  q[1] = 0;
}
// (the limbs of a stored cell are zero: its previous content was consumed)
__device__ __forceinline__ void tab_store(const TrackParams& P, int c, u32 slot, i128 v) {
  u64* q = tab_i128(P, c, slot);
  q[0] = (u64)v;
  q[1] = (u64)((u128)v >> 64);
}

// add cnt members to table slot `slot` (fire-and-forget); the thread whose
// ht_insert created the key appends the slot to the frame's occupied list
__device__ __forceinline__ void touch_cell(const TrackParams& P, TrackCtl* C, u32 slot, u32 cnt,
                                           bool created) {
  atomicAdd(P.tab_cnt + slot, cnt);
  if (created) {
    u32 idx = atomicAdd(&C->n_occ, 1u);
    if (idx < (u32)MAXM) P.occ[idx] = slot;
  }
}



// ===========================================================================
// pcSIR step 1
// ===========================================================================
// v - ref exactly representable (TwoSum error 0) and |v - ref| < 128
__device__ __forceinline__ bool delta_exact(float v, float ref, float& s) {
  s = __fsub_rn(v, ref);
  float bp = __fsub_rn(s, v);
  float ap = __fsub_rn(s, bp);
  float err = __fadd_rn(__fsub_rn(v, ap), __fsub_rn(-ref, bp));
  return err == 0.0f && fabsf(s) < 128.0f;
}


// table slot of flat cell id `flat` in the hash-key array (ht_insert without
// the TrackParams, for the out-of-line cell flush)
__device__ __forceinline__ u32 ht_insert_k(u32* hkey, u32 flat, int sh, bool& created) {
  created = false;
  u32 s = ht_hash(flat, sh);
  for (u32 probe = 0; probe < HT_CAP; ++probe) {
    const u32 k = __ldcg(hkey + s);
    if (k == flat) return s;
    if (k == HT_EMPTY) {
      const u32 old = atomicCAS(hkey + s, HT_EMPTY, flat);
      created = (old == HT_EMPTY);
      if (old == HT_EMPTY || old == flat) return s;
    }
    s = (s + 1) & (HT_CAP - 1);
  }
  return HT_EMPTY;
}

// shared-memory slot of sub-window cell q in the per-cell accumulators: a
// permutation inside each row of 32 cells so that a compact blob of cells
// (the particle cloud) spreads over all 32 banks instead of one bank per
// column (bank conflicts of the shared atomics)
__device__ __forceinline__ int s1_swz(int q) { return (q & ~31) | ((q + 13 * (q >> 5)) & 31); }

// the exact int128 value of the three 16/16/signed digit accumulators of
// component c, cell q (S1Smem.dig)
__device__ __forceinline__ i128 s1_digits(u32 d0, u32 d1, u32 d2) {
  return (i128)d0 + ((i128)d1 << 16) + ((i128)(int)d2 << 32);
}

// Out-of-line partial flush of ONE sub-window cell whose member count just
// crossed a multiple of S1_CELL_FLUSH: each digit is taken with an atomic
// exchange (additions racing with it land either in the taken value or in
// the accumulator, never in both), so no other warp has to stop. The count
// and the cell-edge offsets stay for the final flush.
__device__ __noinline__ void s1_cell_flush(u32* dig, int q, u32 flat, u32* hkey, int ht_shift,
                                           u64* tab_sum, i64 G, u32* occ, TrackCtl* C) {
  i128 s[5];
#pragma unroll
  for (int c = 0; c < 5; ++c) {
    const u32 d0 = atomicExch(dig + (3 * c) * SUBW + q, 0u);
    const u32 d1 = atomicExch(dig + (3 * c + 1) * SUBW + q, 0u);
    const u32 d2 = atomicExch(dig + (3 * c + 2) * SUBW + q, 0u);
    s[c] = s1_digits(d0, d1, d2);
  }
  bool created;
  const u32 slot = ht_insert_k(hkey, flat, ht_shift, created);
  if (slot == HT_EMPTY) {
    set_flag(C, PCS_FLAG_CAPACITY);
    return;
  }
  atomic_add_i128_x5(tab_sum + (i64)slot * 2, G * 2, s);
  if (created) {
    const u32 idx = atomicAdd(&C->n_occ, 1u);
    if (idx < (u32)MAXM) occ[idx] = slot;
  }
  atomicAdd(&C->s1_mid_flush, 1u);
}

// fold the CTA's accumulators (digits + count + cell-edge offsets) into the
// exact int128 HBM table (after the CTA's last particle)
__device__ __forceinline__ void s1_flush(const TrackParams& P, TrackCtl* C, S1Smem& sm, i64 sx0,
                                         i64 sy0, int snx, int sny) {
  const Grid& g = P.grid;
  for (int q = threadIdx.x; q < snx * sny; q += S1_THREADS) {
    const int qs = s1_swz(q);
    const u32 cnt = sm.cnt[qs];
    if (cnt == 0) continue;
    const int qx = q % snx, qy = q / snx;
    const u32 flat = (u32)((sy0 + qy) * g.ncols + (sx0 + qx));
    i128 s[5];
#pragma unroll
    for (int c = 0; c < 5; ++c)
      s[c] = s1_digits(sm.dig[3 * c][qs], sm.dig[3 * c + 1][qs], sm.dig[3 * c + 2][qs]);
    s[0] += (i128)cnt * f32_to_fixed(sm.ref[qx], FX_STATE);
    s[1] += (i128)cnt * f32_to_fixed(sm.ref[snx + qy], FX_STATE);
    bool created;
    const u32 slot = ht_insert(P, flat, created);
    if (slot != HT_EMPTY) {
      atomic_add_i128_x5(P.tab_sum + (i64)slot * 2, P.G * 2, s);
      touch_cell(P, C, slot, cnt, created);
    } else {
      set_flag(C, PCS_FLAG_CAPACITY);
    }
  }
}

// add one in-window particle's exact values (x - ref, y - ref, vx, vy, I0;
// round(v 2^40) exact, |v| < 128) to cell q: the int64 V splits into bits
// 0-15, 16-31 (unsigned) and V >> 32 (signed, |.| < 2^15), each added with a
// native 32-bit shared atomic
__device__ __forceinline__ void s1_add(u32* dig, int q, const float (&v)[5]) {
#pragma unroll
  for (int c = 0; c < 5; ++c) {
    const long long V = __float2ll_rn(__fmul_rn(v[c], 1099511627776.0f));
    const u32 lo = (u32)V;
    atomicAdd(dig + (3 * c) * SUBW + q, lo & 0xFFFFu);
    atomicAdd(dig + (3 * c + 1) * SUBW + q, lo >> 16);
    atomicAdd(dig + (3 * c + 2) * SUBW + q, (u32)(V >> 32));
  }
}

// QUEUE: the instantiation for the first frame of a track (the initial cloud
// is usually wider than the sub-window): particles outside it are queued per
// warp and handled 32 at a time; the steady-state instantiation handles the
// few there are on the spot.
template <bool POW2, bool QUEUE = false>
__global__ void __launch_bounds__(S1_THREADS, S1_CTAS_PER_SM) k_pc_step1(TrackParams P) {
  extern __shared__ __align__(16) unsigned char s1_raw[];
  S1Smem& sm = *reinterpret_cast<S1Smem*>(s1_raw);
  S1Queue& sq = *reinterpret_cast<S1Queue*>(s1_raw + (QUEUE ? sizeof(S1Smem) : 0));   // (QUEUE only)
  TrackCtl* C = P.ctl;
  pdl_trigger();
  if (C->flags & PCS_FLAG_CAPACITY) return;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  if (blockIdx.x == 0 && t == 0) C->pc_prior = C->prior_nonuniform;   // read after this kernel
  const i64 k = C->k;
  const float* sin = (k & 1) ? P.buf1 : P.buf0;
  float* sout = (k & 1) ? P.buf0 : P.buf1;
  const Grid g = P.grid;
  const i64 n = P.n, ld = P.ld;

  // sub-window (identical in every CTA): centred on the previous estimate
  i64 snx = min((i64)S1_SIDE, g.ncols), sny = min((i64)S1_SIDE, g.nrows);
  if (snx < S1_SIDE) sny = min(g.nrows, (i64)(SUBW / snx));
  if (sny < S1_SIDE) snx = min(g.ncols, (i64)(SUBW / sny));
  i64 cx = cell_axis_fast((float)C->center[0], g.ox, g.lx, P.inv_lx, g.ncols);
  i64 cy = cell_axis_fast((float)C->center[1], g.oy, g.ly, P.inv_ly, g.nrows);
  const i64 sx0 = min(max(cx - snx / 2, (i64)0), g.ncols - snx);
  const i64 sy0 = min(max(cy - sny / 2, (i64)0), g.nrows - sny);
  if (blockIdx.x == 0 && t == 0) {
    C->sx0 = sx0; C->sy0 = sy0; C->snx = snx; C->sny = sny;
  }
  const int snxi = (int)snx, snyi = (int)sny;
  for (int q = t; q < SUBW; q += S1_THREADS) {
    sm.cnt[q] = 0;
#pragma unroll
    for (int p = 0; p < S1_PARTS; ++p) sm.dig[p][q] = 0;
  }
  // cell lower edges; NaN marks an edge whose deltas may not be exact.
  // fast_delta: every edge r of the sub-window is >= 2 l (and l < 64), so for
  // any x of the cell, r/2 <= x <= 2r and x - r is exact (Sterbenz) — no
  // TwoSum check per particle
  if (QUEUE && t < S1_WARPS) sq.oqn[t] = 0;
  if (t == 0) {
    sm.fast_delta = (g.lx < 64.0 && g.ly < 64.0) ? 1 : 0;
    sm.fl_hkey = P.hkey;
    sm.fl_shift = P.ht_shift;
    sm.fl_tab_sum = P.tab_sum;
    sm.fl_occ = P.occ;
    sm.fl_G = P.G;
  }
  __syncthreads();
  for (int q = t; q < snxi + snyi; q += S1_THREADS) {
    bool ok;
    float r = (q < snxi) ? cell_ref32(g.ox, g.lx, sx0 + q, ok)
                         : cell_ref32(g.oy, g.ly, sy0 + (q - snxi), ok);
    sm.ref[q] = ok ? r : __int_as_float(0x7fc00000);
    const double l2 = 2.0 * ((q < snxi) ? g.lx : g.ly);
    if (!ok || !((double)r >= l2)) atomicAnd(&sm.fast_delta, 0);
  }
  const float* refy = sm.ref + snxi;
  __syncthreads();
  const bool fast_delta = sm.fast_delta != 0;

  const u32 frame = P.frame0 + (u32)k;
  const AxisFast& axx = P.axx;   // (host-computed: constant-bank operands, no registers)
  const AxisFast& axy = P.axy;
  const u32 ncols32 = (u32)g.ncols;
  const int sx0i = (int)sx0, sy0i = (int)sy0;
  u32* dig = &sm.dig[0][0];
  bool bad = false;
  // warp tiles of P.s1_tile particles (sized by the host so that every warp
  // gets the same number); the first is static, later ones come from a
  // ticket counter drawn one tile ahead (warps on slower SMs take fewer).
  // Each warp streams its tiles as chunks of S1_CHUNK particles; the next
  // chunk's ancestor indices are loaded while the current chunk computes.
  const int WT = P.s1_tile;
  const int nwarps = (int)gridDim.x * S1_WARPS;
  const int ntile = (int)ceil_div(n, (i64)WT);
  u32 tk = 0;   // (lane 0) the ticket of the tile after the latest one entered
  if (lane == 0) tk = atomicAdd(&C->s1_ticket, 1u);
  auto first_chunk = [&](int tl, int& jb, int& je) {
    if (tl < ntile) {
      jb = tl * WT;
      je = (int)min((i64)jb + WT, n);
    } else {
      jb = -1;
      je = 0;
    }
  };
  auto next_chunk = [&](int& jb, int& je) {
    if (jb < 0) return;
    jb += S1_CHUNK;
    if (jb < je) return;
    const int tl = nwarps + (int)__shfl_sync(0xffffffffu, tk, 0);
    if (lane == 0 && tl < ntile) tk = atomicAdd(&C->s1_ticket, 1u);
    first_chunk(tl, jb, je);
  };
  auto load_src = [&](int jb, int je, int (&src)[S1_IPT]) {
#pragma unroll
    for (int it = 0; it < S1_IPT; ++it) {
      const int j = jb + it * 32 + lane;
      src[it] = (jb >= 0 && j < je) ? __ldg(P.anc + j) : -1;
    }
  };
  int jb0, je0, jb1, je1;
  first_chunk((int)blockIdx.x * S1_WARPS + warp, jb0, je0);
  jb1 = jb0; je1 = je0; next_chunk(jb1, je1);
  int src_k[S1_IPT], src1[S1_IPT];
  float o_k[S1_IPT][5];
  // component base pointers (warp-uniform): one 64-bit offset per particle,
  // no per-component pointer steps; an unused lane loads particle 0
  const float* sinc[5];
  float* soutc[5];
#pragma unroll
  for (int c = 0; c < 5; ++c) {
    sinc[c] = sin + c * ld;
    soutc[c] = sout + c * ld;
  }
  auto load_states = [&](const int (&src)[S1_IPT], float (&o)[S1_IPT][5]) {
#pragma unroll
    for (int it = 0; it < S1_IPT; ++it) {
      const u32 sj = (u32)max(src[it], 0);
#pragma unroll
      for (int c = 0; c < 5; ++c) o[it][c] = __ldg(sinc[c] + sj);
    }
  };
  // queued particles (outside cells): exact fire-and-forget limb reductions
  // straight to the cell's table slot, one particle per lane; whole batches
  // of 32 (all of them when `all`), the rest moves to the front of the queue.
  // The state values are read back from this frame's output (written by this
  // warp; the warp barrier orders them).
  // a particle outside the shared sub-window: exact fire-and-forget limb
  // reductions straight to its cell's table slot (jw: particle index, bit 31
  // = its cell code is already written)
  auto outside_cell = [&](u32 flat, u32 jw, const float* v) {
    bool created;
    const u32 slot = ht_insert(P, flat, created);
    if (!(jw & 0x80000000u)) __stcs(P.pslot + (jw & 0x7FFFFFFFu), (u32)SUBW + slot);   // its cell code
    if (slot != HT_EMPTY) {
#pragma unroll
      for (int c = 0; c < 5; ++c) tab_add_f32(tab_ptr(P, c, slot), v[c]);
      touch_cell(P, C, slot, 1u, created);
    } else {
      set_flag(C, PCS_FLAG_CAPACITY);
    }
  };
  constexpr bool use_q = QUEUE;
  auto drain_outside = [&](bool all) {
    __syncwarp();
    const int qn = (int)sq.oqn[warp];
    if (qn < 32 && !(all && qn > 0)) return;   // (warp-uniform)
    int done = 0;
    while (qn - done >= 32 || (all && done < qn)) {
      if (done + lane < qn) {
        const u32 flat = sq.oq[warp][done + lane][0], jw = sq.oq[warp][done + lane][1];
        const u32 pj = jw & 0x7FFFFFFFu;
        float v[5];
#pragma unroll
        for (int c = 0; c < 5; ++c) v[c] = __ldcg(soutc[c] + pj);
        outside_cell(flat, jw, v);
      }
      done += 32;
    }
    done = min(done, qn);
    const int left = qn - done;
    u32 e0 = 0, e1 = 0;
    if (lane < left) {
      e0 = sq.oq[warp][done + lane][0];
      e1 = sq.oq[warp][done + lane][1];
    }
    __syncwarp();
    if (lane < left) {
      sq.oq[warp][lane][0] = e0;
      sq.oq[warp][lane][1] = e1;
    }
    if (lane == 0) sq.oqn[warp] = (u32)left;
    __syncwarp();
  };
  load_src(jb0, je0, src_k);
#if PCS_S1_DEEP
  load_states(src_k, o_k);
  load_src(jb1, je1, src1);
#endif
  while (jb0 >= 0) {
#if PCS_S1_DEEP
    // the next chunk's states (its ancestors arrived during the last chunk)
    // and the ancestors of the one after move while this chunk computes
    float o_n[S1_IPT][5];
    load_states(src1, o_n);
    int jb2 = jb1, je2 = je1;
    next_chunk(jb2, je2);
    int src2[S1_IPT];
    load_src(jb2, je2, src2);
#else
    load_src(jb1, je1, src1);   // the next chunk's ancestors (consumed next iteration)
    load_states(src_k, o_k);
#endif
#pragma unroll
    for (int it = 0; it < S1_IPT; ++it) {
      if (src_k[it] < 0) continue;
      const int j = jb0 + it * 32 + lane;
      float s[5], z[5];
#pragma unroll
      for (int c = 0; c < 5; ++c) s[c] = o_k[it][c];
      philox_normals5k(P.pk, frame, (u64)(P.idx_off + j), z);
      float* o = o_k[it];
      propagate_one(s, z, P.dyn, o);
#pragma unroll
      for (int c = 0; c < 5; ++c) __stcs(soutc[c] + (u32)j, o[c]);   // (read next frame: > L2)
      if (!(o[0] == o[0]) || !(o[1] == o[1])) bad = true;
      const int ix = cell_axis_hot<POW2>(o[0], axx);
      const int iy = cell_axis_hot<POW2>(o[1], axy);
      const u32 flat = (u32)iy * ncols32 + (u32)ix;   // G <= 2^32 - 1
      const int lx = ix - sx0i, ly = iy - sy0i;
      const bool inwin = (u32)lx < (u32)snxi && (u32)ly < (u32)snyi;
      if (inwin) __stcs(P.pslot + j, (u32)(ly * snxi + lx));   // cell code (else: below)
      float dx, dy;
      bool dok = false;
      if (inwin) {
        if (fast_delta) {   // (CTA-uniform branch)
          dx = __fsub_rn(o[0], sm.ref[lx]);
          dy = __fsub_rn(o[1], refy[ly]);
          dok = true;
        } else {
          dok = delta_exact(o[0], sm.ref[lx], dx) && delta_exact(o[1], refy[ly], dy);
        }
      }
      if (dok && fabsf(o[2]) < 128.0f && fabsf(o[3]) < 128.0f && fabsf(o[4]) < 128.0f) {
        const int qs = s1_swz(ly * snxi + lx);
        const u32 old = atomicAdd(&sm.cnt[qs], 1u);
        if (((old + 1u) & (S1_CELL_FLUSH - 1u)) == 0u)
          s1_cell_flush(dig, qs, flat, sm.fl_hkey, sm.fl_shift, sm.fl_tab_sum, sm.fl_G, sm.fl_occ, C);
        o[0] = dx;
        o[1] = dy;
        s1_add(dig, qs, o_k[it]);
      } else {
        // outside the shared sub-window (frame 0 of a track: ~9 % of the wide
        // initial cloud), or values beyond the digit range: queued per warp
        // and handled 32 at a time at the end of the chunk, instead of every
        // warp iteration running that path for two or three lanes. The
        // lanes here together reserve their entries (warp-aggregated atomic).
        if (use_q) {   // (CTA-uniform)
          const unsigned m = __activemask();
          const int leader = __ffs(m) - 1;
          u32 qb = 0;
          if (lane == leader) qb = atomicAdd(&sq.oqn[warp], (u32)__popc(m));
          qb = __shfl_sync(m, qb, leader) + (u32)__popc(m & ((1u << lane) - 1u));
          sq.oq[warp][qb][0] = flat;
          sq.oq[warp][qb][1] = (u32)j | (inwin ? 0x80000000u : 0u);
        } else {
          outside_cell(flat, (u32)j | (inwin ? 0x80000000u : 0u), o);
        }
      }
    }
    if (use_q) drain_outside(false);
    jb0 = jb1; je0 = je1;
#if PCS_S1_DEEP
    jb1 = jb2; je1 = je2;
#pragma unroll
    for (int it = 0; it < S1_IPT; ++it) {
      src_k[it] = src1[it];
      src1[it] = src2[it];
#pragma unroll
      for (int c = 0; c < 5; ++c) o_k[it][c] = o_n[it][c];
    }
#else
#pragma unroll
    for (int it = 0; it < S1_IPT; ++it) src_k[it] = src1[it];
    next_chunk(jb1, je1);
#endif
  }
  if (use_q) drain_outside(true);
  __syncthreads();
  if (t == 0 && atomicAdd(&C->s1_done, 1u) == gridDim.x - 1) {   // every ticket is drawn
    C->s1_ticket = 0;
    C->s1_done = 0;
  }
  s1_flush(P, C, sm, sx0, sy0, snxi, snyi);
  if (bad) set_flag(C, PCS_FLAG_NONFINITE);
}

// ===========================================================================
// pcSIR bins (one CTA): dummies, likelihood per occupied cell ((cell, row)
// parallel), normaliser, per-cell weights, estimate, ESS, resampling
// decision. Zeroes the consumed table cells. Latency-bound by design (a few
// hundred cells): everything per cell stays in shared memory, each exact
// reduction is warp shuffles + one barrier + a warp-parallel final sum, and
// the control-block reads of the epilogue are issued at kernel entry.
// ===========================================================================
// ---- TMA staging of frame regions (cp.async.bulk.tensor.3d + mbarrier) ----
constexpr int FMAP_BX = 64, FMAP_BY = 16;   // box = 64 x 16 float32 pixels (4 KB)

__device__ __forceinline__ void tma_frame_box(float* dst, const void* fmap, int x, int y, int z,
                                              unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"((u32)__cvta_generic_to_shared(dst)),
      "l"(fmap), "r"(x), "r"(y), "r"(z), "r"((u32)__cvta_generic_to_shared(bar))
      : "memory");
}

// Stage rows [y0, y0 + 16 nb) x columns [x0, x0 + 64) of frame z into dst
// (pitch 64; out-of-frame pixels arrive as zeros and are never read; x0 must
// be a multiple of 4: box origins are 16-byte aligned, tools/tma_probe.cu).
// One thread arms the mbarrier and issues the nb box copies; every thread waits.
// issue (thread 0 only)
__device__ __forceinline__ void tma_stage_issue(float* dst, const void* fmap, int x0, int y0, int z,
                                                int nb, unsigned long long* bar) {
  const u32 b = (u32)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b),
               "r"((u32)(nb * FMAP_BX * FMAP_BY * 4)) : "memory");
  for (int j = 0; j < nb; ++j)
    tma_frame_box(dst + j * FMAP_BX * FMAP_BY, fmap, x0, y0 + j * FMAP_BY, z, bar);
}
// wait (every thread; after a barrier that orders it behind the issue)
__device__ __forceinline__ void tma_stage_wait(unsigned long long* bar) {
  // try_wait with a suspend-time hint: waiting warps sleep instead of spinning
  // on issue slots the co-resident CTA needs
  asm volatile(
      "{\n\t.reg .pred p;\n\tTMA_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0, %1;\n\t"
      "@!p bra TMA_WAIT_%=;\n\t}" ::"r"((u32)__cvta_generic_to_shared(bar)), "r"(1000000u) : "memory");
}

// per-cell records of the frame's occupied cells (global memory, MAXM each)
struct BinsScratch {
  double* ll;    // cell log-likelihood, then exp(ll - max) (k_pc_bins)
  u32* cnt;      // members
};

// ---------------------------------------------------------------------------
// k_pc_cells: one warp per occupied cell, all SMs — the dummy (exact mean,
// binning.py:157-172; weighted centre of mass with uniform prior weights;
// cell centre, :168-171) and its likelihood (binning.py:189), the Gaussian
// SSD in the canonical float32 form (identical to SIR on one-particle
// cells), the Poisson models in float64 (pcs_lik.cuh loglik_poisson64_warp).
// Publishes ll and count per cell and the frame's largest log-likelihood.
// ---------------------------------------------------------------------------
constexpr int CELLS_BLOCK = 256;

__global__ void __launch_bounds__(CELLS_BLOCK) k_pc_cells(TrackParams P, BinsScratch Sd) {
  TrackCtl* C = P.ctl;
  pdl_wait();
  pdl_trigger();   // the bins kernel may be scheduled
  const u32 nocc = C->n_occ;
  if ((C->flags & PCS_FLAG_CAPACITY) || nocc > (u32)MAXM) return;   // (k_pc_bins reports it)
  const int M = (int)nocc;
  const int lane = threadIdx.x & 31;
  const i64 k = C->k;
  const float* frame = C->frames + (k - C->k_frames) * P.H * P.W;
  const PixView pv = frame_view(frame, P.H, P.W);
  const bool f64 = P.spot.model != 0 && P.spot.f64;
  const u64 wq0 = P.weighted ? (u64)f32_to_fixed(__double2float_rn(__ddiv_rn(1.0, (double)P.n_global)), FX_WQ)
                             : 0ull;
  long long lmax = LLONG_MIN;
  const int nw = gridDim.x * (CELLS_BLOCK / 32);
  for (int b = blockIdx.x * (CELLS_BLOCK / 32) + (threadIdx.x >> 5); b < M; b += nw) {
    const u32 cell = P.occ[b];
    const u32 cnt = P.tab_cnt[cell];
    // dummy x, y, I0 (vx, vy do not enter the likelihood); weighted centre
    // of mass with the general path's uniform prior weight w0 = RN32(1/N):
    // RN32(RN64(RN64(wq S) / RN64(wq count)) 2^-40), wq = round(w0 2^62)
    const double den = P.weighted ? i128_to_f64_rn((i128)wq0 * (i128)cnt) : (double)cnt;
    // fold the cell's limb sums into its int128 sums (lane c: component c), so
    // the bins kernel reads one exact sum per component
    i128 Sc = 0;
    if (lane < 5) {
      Sc = tab_load(P, lane, cell);
      u64* q = tab_i128(P, lane, cell);
      q[0] = (u64)Sc;
      q[1] = (u64)((u128)Sc >> 64);
      u64* l = tab_ptr(P, lane, cell);
      l[0] = 0;
      l[1] = 0;
      l[2] = 0;
    }
    float d[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int c = (q == 2) ? 4 : q;
      const u64 lo = __shfl_sync(0xffffffffu, (u64)Sc, c);
      const u64 hi = __shfl_sync(0xffffffffu, (u64)((u128)Sc >> 64), c);
      const i128 S = (i128)(((u128)hi << 64) | (u128)lo);
      const double num = i128_to_f64_rn(P.weighted ? S * (i128)wq0 : S);
      d[q] = __double2float_rn(scalbn(__ddiv_rn(num, den), -FX_STATE));
    }
    if (P.placement == 1) {   // cell centre (binning.py:168-171)
      const u32 flat = P.hkey[cell];
      const i64 ix = (i64)flat % P.grid.ncols, iy = (i64)flat / P.grid.ncols;
      d[0] = __double2float_rn(__dadd_rn(P.grid.ox, __dmul_rn((double)ix + 0.5, P.grid.lx)));
      d[1] = __double2float_rn(__dadd_rn(P.grid.oy, __dmul_rn((double)iy + 0.5, P.grid.ly)));
    }
    double ll;
    if (f64) {
      ll = loglik_poisson64_warp(pv, d[0], d[1], d[2], P.spot, lane);
    } else {
      ll = loglik_warp(pv, d[0], d[1], d[2], P.spot, lane);
    }
    if (lane == 0) {
      Sd.ll[b] = ll;
      Sd.cnt[b] = cnt;
      lmax = max(lmax, (long long)f64_to_ordered(ll));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lmax = max(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
  if (lane == 0 && lmax != LLONG_MIN) atomicMax((long long*)&C->cell_max_ord, lmax);
}

constexpr int BINS_BLOCK = 512;
#define PCS_PROBE(i)                                                                  \
  do {                                                                                \
    if (threadIdx.x == 0) {                                                           \
      unsigned long long _g;                                                          \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_g));                          \
      C->dbg[i] = (long long)_g;                                                      \
    }                                                                                 \
  } while (0)

// K exact sums over the block: warp shuffles, one barrier, then warp 0 sums
// the 32 warp partials with shuffles; the results are valid in warp 0
template <int K>
__device__ __forceinline__ void bins_sum_k(i128 (&v)[K], i128* sh) {
#pragma unroll
  for (int c = 0; c < K; ++c) v[c] = warp_sum_i128(v[c]);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) {
#pragma unroll
    for (int c = 0; c < K; ++c) sh[w * K + c] = v[c];
  }
  __syncthreads();
  if (w == 0) {
#pragma unroll
    for (int c = 0; c < K; ++c) v[c] = warp_sum_i128((l < BINS_BLOCK / 32) ? sh[l * K + c] : (i128)0);
  }
}

// ---------------------------------------------------------------------------
// k_pc_bins (one CTA): from the per-cell log-likelihoods of k_pc_cells the
// exact normaliser, per-cell weights (broadcast tables for the resampler),
// estimate, ESS and the resampling decision (filtering.py:75-114,169-170);
// zeroes the consumed table cells. Any number of occupied cells up to MAXM.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(BINS_BLOCK) k_pc_bins(TrackParams P, BinsScratch Sd) {
  TrackCtl* C = P.ctl;
  pdl_wait();
  pdl_trigger();   // k_sys_resample CTAs may become resident on the other SMs
  PCS_PROBE(8);
  __shared__ i128 red[BINS_BLOCK / 32 * 6];
  __shared__ unsigned s_wmin, s_wmax;
  __shared__ double s_Sf;
  const int t = threadIdx.x;
  const i64 k = C->k;
  const u32 nocc = C->n_occ;
  if (t == 0) atomicMax(&C->max_occ, nocc);
  // (weighted centre of mass with non-uniform prior weights needs the
  // per-particle weighted sums of the general path)
  if ((C->flags & PCS_FLAG_CAPACITY) || nocc > (u32)MAXM || (P.weighted && C->pc_prior)) {
    if (t == 0) {
      set_flag(C, PCS_FLAG_CAPACITY);
      C->do_resample = 0;
      // no per-particle finish of this frame: the prior-weight kernels
      // (k_pc_prior_ll, k_sir_sum, k_sir_stats) must not finalise it again
      C->pc_prior = 0;
      C->prior_nonuniform = 0;
      if (k < C->k_end) C->out_occ[k - C->k_out] = -1;
      reset_frame(C);
      C->k = k + 1;
    }
    return;
  }
  const int M = (int)nocc;
  // epilogue inputs, read now so that their latency overlaps the work
  i64 ko = 0;
  double* out_est = nullptr;
  double* out_ess = nullptr;
  unsigned char* out_res = nullptr;
  i64* out_occ = nullptr;
  double u_next = 0.0;
  i64 evals = 0;
  if (t == 0) {
    evals = C->evals;
    ko = k - C->k_out;
    out_est = C->out_est;
    out_ess = C->out_ess;
    out_res = C->out_res;
    out_occ = C->out_occ;
    u_next = philox_resample_u(P.seed, P.frame0 + (u32)k);
    s_wmin = 0xFFFFFFFFu;
    s_wmax = 0u;
  }
  const double m = ordered_to_f64(C->cell_max_ord);
  const bool bad_m = !(m == m) || m == INFINITY;
  const bool degenerate = (m == -INFINITY);
  PCS_PROBE(3);
  if (C->pc_prior) {
    // particles carry prior weights (no resampling at the previous frame):
    // publish the per-cell log-likelihood; the per-particle weights
    // log w = log w_prev + ll_cell (binning.py:190-192), normaliser, estimate,
    // ESS and decision follow in k_pc_prior_ll / k_sir_sum / k_sir_stats
    for (int b = t; b < M; b += BINS_BLOCK) {
      const u32 cell = P.occ[b];   // (table slot)
      const double llb = Sd.ll[b];
      P.lltab[cell] = llb;
      const int qs = sub_code(P, C, P.hkey[cell]);
      if (qs >= 0) P.ltsub[qs] = llb;
      P.hkey[cell] = HT_EMPTY;   // (no kernel probes the table until the next frame)
#pragma unroll
      for (int c = 0; c < 5; ++c) {   // (the limbs were folded by k_pc_cells)
        u64* q = tab_i128(P, c, cell);
        q[0] = 0;
        q[1] = 0;
      }
      P.tab_cnt[cell] = 0;
    }
    if (t == 0) {
      C->frame_occ = M;
      C->cell_max_ord = LLONG_MIN;
    }
    return;
  }
  // normaliser S = sum_b cnt_b * round(exp(ll_b - m) * 2^95)
  {
    i128 acc[1] = {0};
    for (int b = t; b < M; b += BINS_BLOCK) {
      const double ex = exp(__dsub_rn(Sd.ll[b], m));
      Sd.ll[b] = ex;   // the weights below reuse exp(ll - m)
      acc[0] += (i128)Sd.cnt[b] * f64_to_fixed(ex, FX_S);
    }
    bins_sum_k<1>(acc, red);
    if (t == 0) s_Sf = i128_to_f64_scaled(acc[0], FX_S);
    __syncthreads();
  }
  const double Sf = s_Sf;
  PCS_PROBE(4);
  // weights per cell (broadcast tables), estimate, ESS; zero consumed cells
  i128 e[6] = {0, 0, 0, 0, 0, 0};
  {
    unsigned wmin = 0xFFFFFFFFu, wmax = 0u;
    for (int b = t; b < M; b += BINS_BLOCK) {
      const u32 cell = P.occ[b];   // (table slot)
      const u32 cnt = Sd.cnt[b];
      const u32 flat = P.hkey[cell];
      // the cell's state sums first: their latency overlaps the division
      i128 Ssum[5];
#pragma unroll
      for (int c = 0; c < 5; ++c) Ssum[c] = load_i128(tab_i128(P, c, cell));   // (folded by k_pc_cells)
      const float w = __double2float_rn(__ddiv_rn(Sd.ll[b], Sf));   // normalised_weight
      P.wtab[cell] = w;
      P.wfix[cell] = cdf_fixed(w);
      P.hkey[cell] = HT_EMPTY;   // (no kernel probes the table until the next frame)
      const int qs = sub_code(P, C, flat);
      if (qs >= 0) {
        P.wtsub[qs] = w;
        P.wsub[qs] = cdf_fixed(w);
      }
      wmin = min(wmin, __float_as_uint(w));
      wmax = max(wmax, __float_as_uint(w));
      const long long wq = (long long)f32_to_fixed(w, FX_WQ);   // w <= 1: fits 63 bits
#pragma unroll
      for (int c = 0; c < 5; ++c) {
        e[c] += (i128)wq * Ssum[c];
        u64* q = tab_i128(P, c, cell);
        q[0] = 0;
        q[1] = 0;
      }
      e[5] += (i128)cnt * f64_to_fixed((double)w * (double)w, FX_W2);
      P.tab_cnt[cell] = 0;
    }
    atomicMin(&s_wmin, wmin);
    atomicMax(&s_wmax, wmax);
  }
  PCS_PROBE(5);
  bins_sum_k<6>(e, red);
  PCS_PROBE(6);
  // warp 0 holds the six exact sums in every lane: lane c converts sum c
  double conv = 0.0;
  if (t < 32) {
    const int c = min(t, 5);
    i128 ec = e[0];
#pragma unroll
    for (int q = 1; q < 6; ++q) ec = (c == q) ? e[q] : ec;
    conv = i128_to_f64_scaled(ec, c < 5 ? FX_WQ + FX_STATE : FX_W2);
    if (c == 5) conv = 1.0 / conv;   // ESS
  }
  double est[5];
#pragma unroll
  for (int c = 0; c < 5; ++c) est[c] = __shfl_sync(0xffffffffu, conv, c);
  const double ess = __shfl_sync(0xffffffffu, conv, 5);
  if (t == 0) {
    const bool flag_bad = degenerate || bad_m;
    if (degenerate) set_flag(C, PCS_FLAG_DEGENERATE);
    if (bad_m) set_flag(C, PCS_FLAG_NONFINITE);
    const bool row = k < C->k_end;   // (an output row exists for this frame)
    if (row) {
      for (int c = 0; c < 5; ++c) out_est[ko * 5 + c] = est[c];
      out_ess[ko] = ess;
    }
    const int res = (!flag_bad && ess < P.thresh) ? 1 : 0;   // filtering.py:169-170
    // no resampling with unequal weights -> the next frame starts from these
    // per-cell weights (k_sys_resample<1> writes them per particle)
    C->prior_nonuniform = (!res && !flag_bad && s_wmin != s_wmax) ? 1 : 0;
    if (row) {
      out_res[ko] = (unsigned char)res;
      out_occ[ko] = M;
    }
    C->evals = evals + M;
    C->do_resample = res;
    C->m = m;
    C->Sf = Sf;
    C->u = u_next;
    C->res_frame = P.frame0 + (u32)k;
    if (!flag_bad) {
      C->center[0] = est[0];
      C->center[1] = est[1];
    }
    reset_frame(C);
    C->k = k + 1;   // last reader of k in this frame
  }
  PCS_PROBE(7);
  __syncthreads();
  PCS_PROBE(9);
}

// ===========================================================================
// Single-pass exact-prefix systematic resampling: decoupled look-back over
// tiles (dynamic tile tickets guarantee forward progress; the tile status
// carries a frame tag so nothing is reset between frames).
// KIND 1: weight = wtab[pslot[i]] (pcSIR), KIND 2: from ll[i], m, Sf (SIR).
// ===========================================================================
__device__ __forceinline__ void st_release_u32(u32* p, u32 v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ u32 ld_acquire_u32(const u32* p) {
  u32 v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// ===========================================================================
// first slot at/above the cdf value RN64(Pc) 2^-120 (first_slot_fast(cdf_round(Pc))):
// float64 estimate from the top 64 bits of Pc, |error| <= n (3 2^-53 + 2^-63)
// < eps = n 2^-50, exact path otherwise
__device__ __forceinline__ i64 slot_of_prefix(u128 Pc, double u, i64 ng, double nd, double kappa,
                                              double eps) {
  const double t = fma((double)(u64)(Pc >> 57), kappa, -u);
  const double g = ceil(t);
  const double gap = g - t;
  if (gap > eps && gap < 1.0 - eps && g > 0.0 && g < nd) return (i64)g;
  return first_slot_fast(cdf_round(Pc), u, ng, nd, eps);
}
// the exact path of slot_of_prefix out of line (keeps the unrolled hot loop small)
__device__ __noinline__ i64 slot_of_prefix_slow(u128 Pc, double u, i64 ng, double nd, double eps) {
  return first_slot_fast(cdf_round(Pc), u, ng, nd, eps);
}
// slot_of_prefix - base as int for a tile whose slots lie in [base, base + 2^31)
__device__ __forceinline__ int slot_rel(u128 Pc, double u, i64 ng, double nd, double kappa, double eps,
                                        double based, i64 base) {
  const double t = fma((double)(u64)(Pc >> 57), kappa, -u);
  const double g = ceil(t);
  const double gap = g - t;
  if (gap > eps && gap < 1.0 - eps && g > 0.0 && g < nd) return __double2int_rz(g - based);
  return (int)(slot_of_prefix_slow(Pc, u, ng, nd, eps) - base);
}
__device__ __forceinline__ void sts_u32(u32 addr, int v) {
  asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ int lds_u32(u32 addr) {
  int v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}

// Persistent reduce-then-scan systematic resampling (single GPU, scan_mode 0).
// Each CTA owns a contiguous range of tiles (RS_TILE = 5888 particles). Pass
// 1 sums the exact fixed-point weights of its range; after ONE grid-wide
// barrier every CTA adds up the aggregates of the CTAs before it (its exact
// exclusive prefix); pass 2 re-reads its range tile by tile, emits each
// item's slots and writes the ancestors coalesced. Tiles are streamed into a
// two-buffer shared-memory ring by TMA bulk copies (cp.async.bulk +
// mbarrier), so the next tile is in flight while the current one is
// processed. RS_ITEMS (odd) consecutive items per thread: the odd-stride reads of the
// dense tile are bank-conflict free. Requires every CTA to be co-resident
// (grid = SMs x occupancy, set by the host from the occupancy calculator).
#ifndef PCS_RS_ITEMS
#define PCS_RS_ITEMS 23   // 5888-particle tiles, 3 CTAs / SM (profiles/r2_variants.md)
#define PCS_RS_SCAP 25
#endif
constexpr int RS_ITEMS = PCS_RS_ITEMS;
constexpr int RS_TILE = SCAN_BLOCK * RS_ITEMS;   // 5888
// A tile emits ~RS_TILE slots (+- a few %): the emission stage holds
// RS_SCAP slots per thread so that one chunk covers almost every tile (odd:
// the per-thread stride is bank-conflict free)
constexpr int RS_SCAP = PCS_RS_SCAP;
constexpr int RS_STAGE = SCAN_BLOCK * RS_SCAP;   // 6400
constexpr int RS_KBITS = 13;                     // bits of a tile-local item index
static_assert(RS_TILE <= (1 << RS_KBITS), "tagged run heads hold the item index in RS_KBITS bits");

__device__ __forceinline__ void grid_barrier(TrackCtl* C, int nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const u32 gen = ld_acquire_u32(&C->gbar_gen);
    __threadfence();
    if (atomicAdd(&C->gbar_cnt, 1u) == (u32)nblocks - 1u) {
      C->gbar_cnt = 0;
      __threadfence();
      st_release_u32(&C->gbar_gen, gen + 1u);
    } else {
      while (ld_acquire_u32(&C->gbar_gen) == gen) __nanosleep(64);
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, u32 parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
// one thread: arm the barrier with the byte count and start the bulk copy
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, u32 bytes,
                                            unsigned long long* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// staged element: KIND 1 the particle's cell id, KIND 2 its log-likelihood
template <int KIND> struct RsElem { typedef u32 T; };
template <> struct RsElem<2> { typedef double T; };

// globaltimer stamps of CTA 0 (dbg[10..14]: start, pass 1 done, barrier
// entered, barrier left, prefix done) and the end of the last CTA (dbg[15])
// (diagnostic builds only: -DPCS_RS_PROBE, tools/rs_probe_c5.py)
#ifdef PCS_RS_PROBE
#define RS_PROBE(i)                                                                   \
  do {                                                                                \
    if (threadIdx.x == 0 && (blockIdx.x == 0 || ((i) == 4 && blockIdx.x == gridDim.x - 1))) { \
      unsigned long long _g;                                                          \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_g));                          \
      C->dbg[(i) == 4 && blockIdx.x == gridDim.x - 1 ? 15 : 10 + (i)] = (long long)_g; \
    }                                                                                 \
  } while (0)
#else
#define RS_PROBE(i) do {} while (0)
#endif

template <int KIND>
struct RsSmem {
  typename RsElem<KIND>::T ring[2][RS_TILE];   // TMA ring (16-byte aligned)
  int stage[RS_STAGE];              // (KIND 1 pass 1: the cell-code histogram, SUBW entries)
  int hp[KIND == 1 ? 1 : RS_TILE];   // run heads (KIND 1: in place of the consumed cell ids)
  u128 wtot[SCAN_BLOCK / 32];
  int s_wmax[SCAN_BLOCK / 32];
  long long s_jr[2];
  unsigned long long bar[2];
};

// MULTI: multinomial scheme — write the exact cdf per particle instead of
// emitting slots (k_multinomial_emit draws them); a separate instantiation so
// the systematic kernel carries none of it
template <int KIND, bool MULTI = false>
#ifndef PCS_RS_MINB
#define PCS_RS_MINB 3
#endif
__global__ void __launch_bounds__(SCAN_BLOCK, KIND == 1 ? PCS_RS_MINB : 2) k_sys_resample(TrackParams P) {
  typedef typename RsElem<KIND>::T E;
  extern __shared__ __align__(128) unsigned char rs_raw[];
  RsSmem<KIND>& sm = *reinterpret_cast<RsSmem<KIND>*>(rs_raw);
  auto& ring = sm.ring;
  int* stage = sm.stage;
  int* hp_own = sm.hp;
  u128* wtot = sm.wtot;
  int* s_wmax = sm.s_wmax;
  unsigned long long* bar = sm.bar;
  TrackCtl* C = P.ctl;
  pdl_wait();   // (no early trigger here: the next frame's step 1 must not
                // take SMs that CTAs of this grid-barrier kernel still need)
  const i64 n = P.n;
  const i64 nt = ceil_div(n, (i64)RS_TILE);
  const int G = gridDim.x, cta = blockIdx.x;
  const i64 t0 = nt * cta / G, t1 = nt * (cta + 1) / G;
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  // pcSIR frames with prior weights resample per particle (KIND 2), the others
  // per cell (KIND 1); both are in the frame's launch sequence
  if (KIND == 1 ? C->pc_prior != 0 : (P.method == 1 && C->pc_prior == 0)) return;
  // sharded filter (pcs_shard.cuh): mode 1 = pass 1 only (per-CTA totals ->
  // rank total), mode 2 = pass 2 only, its prefix offset by the exact weight
  // of the preceding ranks and its slots written from the rank's first slot
  const int mode = P.scan_mode;
  if (!C->do_resample) {   // identity ancestors; the particles keep their weights
    if (mode != 0) return;   // (the shard pack kernel installs the identity)
    const bool keep = C->prior_nonuniform;
    const double Sf = C->Sf;
    for (i64 i = t0 * RS_TILE + threadIdx.x; i < min(n, t1 * RS_TILE); i += SCAN_BLOCK) {
      P.anc_out[P.idx_off + i - P.slot_lo] = (int)i;
      if (keep) P.wprev[i] = (KIND == 1) ? code_wtab(P, P.pslot[i]) : weight_from_ex(P.ll[i], Sf);
    }
    return;
  }
  const double m = C->m, Sf = C->Sf, u = C->u;
  RS_PROBE(0);
  const E* src = (KIND == 1) ? (const E*)(const void*)P.pslot : (const E*)(const void*)P.ll;
  const int mt = (int)(t1 - t0);      // tiles of this CTA; loads L = 0..2 mt-1 (two passes)
  const int L0 = (mode == 2) ? mt : 0, Lend = (mode == 1) ? mt : 2 * mt;
  // load L (absolute: tile t0 + L % mt) goes to ring buffer / mbarrier
  // (L - L0) & 1 and completes phase ((L - L0) >> 1) & 1 of that barrier
  auto issue = [&](int L) {           // thread 0 only
    const i64 tile = t0 + (L % mt);
    const i64 b0 = tile * RS_TILE;
    const i64 cnt = min((i64)RS_TILE, n - b0);
    const u32 bytes = (u32)(((cnt * (i64)sizeof(E)) + 15) & ~(i64)15);
    tma_load_1d(ring[(L - L0) & 1], src + b0, bytes, &bar[(L - L0) & 1]);
  };
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0 && mt > 0) issue(L0);
  // exact weight of item k of a ring buffer (nv = valid items of its tile)
  auto weight = [&](const E* buf, int k, int nv) -> u128 {
    if (k >= nv) return 0;
    if (KIND == 1) return code_wfix(P, (u32)buf[k]);
    return cdf_fixed(weight_from_ex((double)buf[k], Sf));
  };
  auto tile_items = [&](i64 tile) -> int { return (int)min((i64)RS_TILE, n - tile * RS_TILE); };
  // ---- pass 1: this CTA's exact total ----
  // KIND 1: a histogram of the sub-window cell codes (one shared atomic per
  // item, bank-swizzled), folded with the exact cell weights at the end;
  // codes of cells outside the sub-window add their weight directly
  u128 acc = 0;
  if (KIND == 1 && mode != 2) {
    static_assert(RS_STAGE >= SUBW, "the pass-1 histogram lives in the emission stage");
    u32* hist = reinterpret_cast<u32*>(sm.stage);
    for (int q = threadIdx.x; q < SUBW; q += SCAN_BLOCK) hist[q] = 0;
    __syncthreads();
    for (int L = 0; L < mt; ++L) {
      mbar_wait(&bar[L & 1], (u32)((L >> 1) & 1));
      if (threadIdx.x == 0 && L + 1 < Lend) issue(L + 1);
      const E* buf = ring[L & 1];
      const int nv = tile_items(t0 + L);
      const int kb = threadIdx.x * RS_ITEMS;
      auto item = [&](int k) {
        const u32 code = (u32)buf[k];
        if (code < (u32)SUBW) atomicAdd(hist + s1_swz((int)code), 1u);
        else acc += P.wfix[code - SUBW];
      };
      if (nv == RS_TILE) {
        // warp-uniform: any cell outside the sub-window in this thread group's
        // items (frame 0 of a track: the wide initial cloud)? then their
        // table weights are fetched by independent predicated loads, not by
        // a divergent load -> add chain per item
        u32 codes[RS_ITEMS];
        bool any_out = false;
#pragma unroll
        for (int q = 0; q < RS_ITEMS; ++q) {
          codes[q] = (u32)buf[kb + q];
          any_out |= codes[q] >= (u32)SUBW;
        }
#pragma unroll
        for (int q = 0; q < RS_ITEMS; ++q)
          if (codes[q] < (u32)SUBW) atomicAdd(hist + s1_swz((int)codes[q]), 1u);
        if (__any_sync(0xffffffffu, any_out)) {
          constexpr int B = 6;   // loads in flight per thread
#pragma unroll
          for (int q0 = 0; q0 < RS_ITEMS; q0 += B) {
            u128 wq[B];
#pragma unroll
            for (int q = 0; q < B; ++q) {
              wq[q] = 0;
              if (q0 + q < RS_ITEMS && codes[q0 + q] >= (u32)SUBW) wq[q] = P.wsub[codes[q0 + q]];
            }
#pragma unroll
            for (int q = 0; q < B; ++q) acc += wq[q];
          }
        }
      } else {
        for (int q = 0; q < RS_ITEMS; ++q)
          if (kb + q < nv) item(kb + q);
      }
      __syncthreads();   // buffer L & 1 is free for load L + 2
    }
    for (int q = threadIdx.x; q < SUBW; q += SCAN_BLOCK) {
      const u32 c = hist[s1_swz(q)];
      if (c) acc += P.wsub[q] * (u128)c;
    }
  } else {
    for (int L = 0; L < (mode == 2 ? 0 : mt); ++L) {   // (L0 == 0 here)
      mbar_wait(&bar[L & 1], (u32)((L >> 1) & 1));
      if (threadIdx.x == 0 && L + 1 < Lend) issue(L + 1);
      const E* buf = ring[L & 1];
      const int nv = tile_items(t0 + L);
#pragma unroll 5
      for (int q = 0; q < RS_ITEMS; ++q) acc += weight(buf, threadIdx.x * RS_ITEMS + q, nv);
      __syncthreads();   // buffer L & 1 is free for load L + 2
    }
  }
  if (mode != 2) {
    u128 v = acc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const u64 lo = (u64)v, hi = (u64)(v >> 64);
      v += ((u128)__shfl_xor_sync(0xffffffffu, hi, o) << 64) | (u128)__shfl_xor_sync(0xffffffffu, lo, o);
    }
    if (lane == 0) wtot[wi] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      u128 tot = 0;
      for (int w = 0; w < SCAN_BLOCK / 32; ++w) tot += wtot[w];
      P.cta_agg[cta] = tot;
      __threadfence();
    }
    if (mode == 1) return;   // (k_shard_total adds the CTA totals)
  }
  RS_PROBE(1);
  if (mode == 0) grid_barrier(C, G);   // (mode 2: the totals come from the mode-1 launch)
  RS_PROBE(2);
  // ---- exclusive prefix of this CTA: aggregates of the CTAs before it ----
  u128 pre;
  {
    u128 v = 0;
    for (int k = threadIdx.x; k < cta; k += SCAN_BLOCK) v += *((volatile u128*)(P.cta_agg + k));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const u64 lo = (u64)v, hi = (u64)(v >> 64);
      v += ((u128)__shfl_xor_sync(0xffffffffu, hi, o) << 64) | (u128)__shfl_xor_sync(0xffffffffu, lo, o);
    }
    if (lane == 0) wtot[wi] = v;
    __syncthreads();
    pre = 0;
    for (int w = 0; w < SCAN_BLOCK / 32; ++w) pre += wtot[w];
    if (mode == 2) pre += ((u128)C->rank_prefix[1] << 64) | (u128)C->rank_prefix[0];
    __syncthreads();
  }
  RS_PROBE(3);
  // ---- pass 2: per tile, item prefixes -> run heads -> ancestors ----
  const i64 ng = P.n_global, off = P.idx_off, cap = P.slot_cap;
  const i64 lo = (mode == 2) ? C->shard_lo : P.slot_lo;
  const double nd = (double)ng, eps = nd * 8.881784197001252e-16;   // n * 2^-50
  const double kappa = nd * 1.0842021724855044e-19;                  // n * 2^-63
  bool oob = false;
  const int k0 = (int)threadIdx.x * RS_ITEMS;
  i64 tj_prev = 0;
  // nothing left in the stage (pass-1 histogram, an earlier launch) may pass
  // for a tagged run head (ordered before the first heads by the first
  // tile's barrier)
  for (int q = threadIdx.x; q < RS_STAGE; q += SCAN_BLOCK) stage[q] = 0;
  for (int L = mt; L < 2 * mt; ++L) {
    const int LL = L - L0;   // load index in this launch
    mbar_wait(&bar[LL & 1], (u32)((LL >> 1) & 1));
    if (threadIdx.x == 0 && L + 1 < Lend) issue(L + 1);
    const E* buf = ring[LL & 1];
    int* hp = (KIND == 1) ? reinterpret_cast<int*>(ring[LL & 1]) : hp_own;
    const i64 base = (t0 + (L - mt)) * RS_TILE;
    const int nv = tile_items(t0 + (L - mt));
    // local index of the globally last item (its run ends at slot ng), -1 if not here
    const i64 kl = ng - 1 - off - base;
    const int klast = (kl >= 0 && kl < nv) ? (int)kl : -1;
    const bool full = (nv == RS_TILE);   // (every tile but the last: no per-item bounds)
    u128 tsum = 0;
    if (full) {
#pragma unroll
      for (int q = 0; q < RS_ITEMS; ++q) tsum += weight(buf, k0 + q, RS_TILE + 1);
    } else {
#pragma unroll 5
      for (int q = 0; q < RS_ITEMS; ++q) tsum += weight(buf, k0 + q, nv);
    }
    u128 inc = tsum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const u128 o = shfl_up_u128(inc, d);
      if (lane >= d) inc += o;
    }
    if (lane == 31) wtot[wi] = inc;
    __syncthreads();
    u128 woff = 0, tagg = 0;
#pragma unroll
    for (int w = 0; w < SCAN_BLOCK / 32; ++w) {
      if (w < wi) woff += wtot[w];
      tagg += wtot[w];
    }
    const u128 excl = pre + woff + (inc - tsum);
    // the tile's slot range, computed by every thread (no broadcast barrier);
    // a tile starts where the previous one ended
    if (L == mt) tj_prev = (off + base == 0) ? 0 : first_slot_fast(cdf_round(pre), u, ng, nd, eps);
    const i64 tj0 = tj_prev;
    const i64 tj1 = (klast == nv - 1) ? ng : first_slot_fast(cdf_round(pre + tagg), u, ng, nd, eps);
    tj_prev = tj1;
    // A tile whose slots fit one emission chunk (almost every tile) scatters
    // its run heads straight into the stage, tagged with the tile's ordinal
    // in the upper bits: a tagged head is larger than anything an earlier
    // tile left there, so the block max-scan needs no fill, and slot 0 of a
    // tile always holds a head of this tile. A larger tile takes the chunked
    // path: run head of every item in hp (its first slot relative to tj0, -1
    // if none), then fill -> heads -> block max-scan per chunk.
    const int m_slots = MULTI ? 0 : (int)(tj1 - tj0);   // <= ng < 2^31
    const int tord = L - mt + 1;                          // 1, 2, ... within this launch
    const bool direct = !MULTI && m_slots <= RS_STAGE && tord < (1 << (31 - RS_KBITS));   // (CTA-uniform)
    {
      const u32 emit_s = smem_u32(stage);
      const int tag = tord << RS_KBITS;
      auto emit = [&](int j0, int j1, int k) {   // item k owns slots [j0, j1) of the tile
        if (j1 > j0 && (u32)j0 < (u32)RS_STAGE) sts_u32(emit_s + 4 * j0, tag | k);
      };
      const double tj0d = (double)tj0;
      int jr = 0;
      if (k0 < nv && off + base + k0 != 0) jr = slot_rel(excl, u, ng, nd, kappa, eps, tj0d, tj0);
      u128 run = excl;
      if (MULTI) {   // the exact cdf per particle (filtering.py:94-95)
#pragma unroll
        for (int q = 0; q < RS_ITEMS; ++q) {
          const int k = k0 + q;
          if (k < nv) {
            run += weight(buf, k, nv);
            P.cdf[base + k] = (k == klast) ? 1.0 : cdf_round(run);
          }
        }
      }
      const u32 hp_s = smem_u32(hp + k0);
      if (direct) {
        if (full && klast < 0) {
#pragma unroll
          for (int q = 0; q < RS_ITEMS; ++q) {
            run += weight(buf, k0 + q, RS_TILE + 1);
            const int jend = slot_rel(run, u, ng, nd, kappa, eps, tj0d, tj0);
            emit(jr, jend, k0 + q);
            jr = jend;
          }
        } else {
#pragma unroll 1
          for (int q = 0; q < RS_ITEMS; ++q) {
            const int k = k0 + q;
            if (k < nv) {
              run += weight(buf, k, nv);
              const int jend = (k == klast) ? (int)(ng - tj0) : slot_rel(run, u, ng, nd, kappa, eps, tj0d, tj0);
              emit(jr, jend, k);
              jr = jend;
            }
          }
        }
      } else if (!MULTI) {
        if (full && klast < 0) {
#pragma unroll
          for (int q = 0; q < RS_ITEMS; ++q) {
            run += weight(buf, k0 + q, RS_TILE + 1);
            const int jend = slot_rel(run, u, ng, nd, kappa, eps, tj0d, tj0);
            sts_u32(hp_s + 4 * q, (jend > jr) ? jr : -1);   // (KIND 1: over item k, already read)
            jr = jend;
          }
        } else {
#pragma unroll
          for (int q = 0; q < RS_ITEMS; ++q) {
            const int k = k0 + q;
            int h = -1;   // no slot
            if (k < nv) {
              run += weight(buf, k, nv);
              const int jend = (k == klast) ? (int)(ng - tj0) : slot_rel(run, u, ng, nd, kappa, eps, tj0d, tj0);
              if (jend > jr) h = jr;
              jr = jend;
            }
            sts_u32(hp_s + 4 * q, h);    // (KIND 1: over item k, already read)
          }
        }
        const u32 st_s = smem_u32(stage + threadIdx.x * RS_SCAP);
#pragma unroll
        for (int q = 0; q < RS_SCAP; ++q) sts_u32(st_s + 4 * q, -1);   // first chunk's fill
      }
    }
    __syncthreads();   // every read of ring[L & 1] is done; it is free for load L + 2
    // slots in chunks of RS_STAGE (one chunk for almost every tile): heads,
    // block max-scan, coalesced writes (multinomial: k_multinomial_emit draws
    // the slots)
    int carry = -1;
    const int ks0 = (int)threadIdx.x * RS_SCAP;          // this thread's stage positions
    const u32 stage_s = smem_u32(stage), hp_s = smem_u32(hp + k0), own_s = smem_u32(stage + ks0);
    for (int c0 = 0; c0 < m_slots; c0 += RS_STAGE) {
      int total = -1;
      {
        if (!direct) {
          if (c0 > 0) {
#pragma unroll
            for (int q = 0; q < RS_SCAP; ++q) sts_u32(own_s + 4 * q, -1);
            __syncthreads();
          }
#pragma unroll
          for (int q = 0; q < RS_ITEMS; ++q) {
            const u32 hr = (u32)(lds_u32(hp_s + 4 * q) - c0);   // no head: (u32)(-1 - c0) >= 2^31
            if (hr < (u32)RS_STAGE) sts_u32(stage_s + 4 * hr, k0 + q);
          }
          __syncthreads();
        }
        int tmax = -1;
#pragma unroll
        for (int q = 0; q < RS_SCAP; ++q) tmax = max(tmax, lds_u32(own_s + 4 * q));
        int incl = tmax;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int o = __shfl_up_sync(0xffffffffu, incl, d);
          if (lane >= d) incl = max(incl, o);
        }
        if (lane == 31) s_wmax[wi] = incl;
        int excl_l = __shfl_up_sync(0xffffffffu, incl, 1);
        if (lane == 0) excl_l = -1;
        __syncthreads();
        int prev = carry;
        total = carry;
#pragma unroll
        for (int w = 0; w < SCAN_BLOCK / 32; ++w) {
          if (w < wi) prev = max(prev, s_wmax[w]);
          total = max(total, s_wmax[w]);
        }
        int runm = max(prev, excl_l);
#pragma unroll
        for (int q = 0; q < RS_SCAP; ++q) {
          runm = max(runm, lds_u32(own_s + 4 * q));
          sts_u32(own_s + 4 * q, runm);
        }
        __syncthreads();
      }
      const int kmask = direct ? (1 << RS_KBITS) - 1 : -1;   // (chunked path: plain indices)
      const int cm = min(RS_STAGE, m_slots - c0);
      const i64 w0 = tj0 + c0 - lo;   // output position of the chunk's first slot
      const int ib = (int)base;
      if (w0 >= 0 && w0 + cm <= cap) {   // coalesced: slot t + q * SCAN_BLOCK
        int* dst = P.anc_out + w0;
        const u32 src_s = stage_s + 4 * threadIdx.x;
#pragma unroll
        for (int q = 0; q < RS_SCAP; ++q) {
          const int k = (int)threadIdx.x + q * SCAN_BLOCK;
          if (k < cm) __stcs(dst + k, ib + (lds_u32(src_s + 4 * q * SCAN_BLOCK) & kmask));   // (evict-first)
        }
      } else {
        for (int k = threadIdx.x; k < cm; k += SCAN_BLOCK) {
          const i64 kk = w0 + k;
          if (kk >= 0 && kk < cap) P.anc_out[kk] = ib + (stage[k] & kmask);
          else oob = true;
        }
      }
      carry = total;
      __syncthreads();
    }
    pre += tagg;
  }
  if (oob) set_flag(C, PCS_FLAG_CAPACITY);
  RS_PROBE(4);
}

// Small-N form of k_sys_resample (every CTA owns ONE tile of RSS_TILE
// particles; used when all those CTAs are co-resident, e.g. c1/c2): the tile
// is staged once, its block scan is done before the grid barrier, and the
// run heads / emission follow right after the prefix — no second pass over
// the input. Same exact arithmetic and output as k_sys_resample.
constexpr int RSS_ITEMS = 7;                        // odd: stride-7 reads are conflict-free
constexpr int RSS_TILE = SCAN_BLOCK * RSS_ITEMS;    // 1792

template <int KIND>
struct RssSmem {
  typename RsElem<KIND>::T items[RSS_TILE];
  int hp[RSS_TILE];
  int stage[RSS_TILE];
  u128 wtot[SCAN_BLOCK / 32];
  int s_wmax[SCAN_BLOCK / 32];
  long long s_jr[2];
};

template <int KIND>
__global__ void __launch_bounds__(SCAN_BLOCK, 4) k_sys_resample_small(TrackParams P) {
  typedef typename RsElem<KIND>::T E;
  __shared__ __align__(16) RssSmem<KIND> sm;
  TrackCtl* C = P.ctl;
  pdl_wait();
  const i64 n = P.n;
  const int G = gridDim.x, cta = blockIdx.x;
  const i64 base = (i64)cta * RSS_TILE;
  const int nv = (int)min((i64)RSS_TILE, n - base);
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  // pcSIR frames with prior weights resample per particle (KIND 2), the others
  // per cell (KIND 1); both are in the frame's launch sequence
  if (KIND == 1 ? C->pc_prior != 0 : (P.method == 1 && C->pc_prior == 0)) return;
  if (!C->do_resample) {   // identity ancestors; the particles keep their weights
    const bool keep = C->prior_nonuniform;
    const double Sf = C->Sf;
    for (int k = threadIdx.x; k < nv; k += SCAN_BLOCK) {
      const i64 i = base + k;
      P.anc_out[P.idx_off + i - P.slot_lo] = (int)i;
      if (keep) P.wprev[i] = (KIND == 1) ? code_wtab(P, P.pslot[i]) : weight_from_ex(P.ll[i], Sf);
    }
    return;
  }
  const double m = C->m, Sf = C->Sf, u = C->u;
  RS_PROBE(0);
  const E* src = (KIND == 1) ? (const E*)(const void*)P.pslot : (const E*)(const void*)P.ll;
  for (int k = threadIdx.x; k < nv; k += SCAN_BLOCK) sm.items[k] = src[base + k];
  __syncthreads();
  auto weight = [&](int k) -> u128 {
    if (k >= nv) return 0;
    if (KIND == 1) return code_wfix(P, (u32)sm.items[k]);
    return cdf_fixed(weight_from_ex((double)sm.items[k], Sf));
  };
  const int k0 = (int)threadIdx.x * RSS_ITEMS;
  u128 tsum = 0;
#pragma unroll
  for (int q = 0; q < RSS_ITEMS; ++q) tsum += weight(k0 + q);
  u128 inc = tsum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const u128 o = shfl_up_u128(inc, d);
    if (lane >= d) inc += o;
  }
  if (lane == 31) sm.wtot[wi] = inc;
  __syncthreads();
  u128 woff = 0, tagg = 0;
#pragma unroll
  for (int w = 0; w < SCAN_BLOCK / 32; ++w) {
    if (w < wi) woff += sm.wtot[w];
    tagg += sm.wtot[w];
  }
  if (threadIdx.x == 0) {
    P.cta_agg[cta] = tagg;
    __threadfence();
  }
  RS_PROBE(1);
  grid_barrier(C, G);
  RS_PROBE(2);
  // exclusive prefix of this CTA: aggregates of the CTAs before it
  u128 pre;
  {
    u128 v = 0;
    for (int k = threadIdx.x; k < cta; k += SCAN_BLOCK) v += *((volatile u128*)(P.cta_agg + k));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const u64 lo = (u64)v, hi = (u64)(v >> 64);
      v += ((u128)__shfl_xor_sync(0xffffffffu, hi, o) << 64) | (u128)__shfl_xor_sync(0xffffffffu, lo, o);
    }
    __syncthreads();   // every thread has read sm.wtot
    if (lane == 0) sm.wtot[wi] = v;
    __syncthreads();
    pre = 0;
#pragma unroll
    for (int w = 0; w < SCAN_BLOCK / 32; ++w) pre += sm.wtot[w];
  }
  RS_PROBE(3);
  const i64 ng = P.n_global, off = P.idx_off, lo = P.slot_lo, cap = P.slot_cap;
  const double nd = (double)ng, eps = nd * 8.881784197001252e-16;   // n * 2^-50
  const double kappa = nd * 1.0842021724855044e-19;                  // n * 2^-63
  const i64 kl = ng - 1 - off - base;
  const int klast = (kl >= 0 && kl < nv) ? (int)kl : -1;
  // the tile's slot range, computed by every thread (no broadcast barrier)
  const i64 tj0 = (off + base == 0) ? 0 : first_slot_fast(cdf_round(pre), u, ng, nd, eps);
  const i64 tj1 = (klast == nv - 1) ? ng : first_slot_fast(cdf_round(pre + tagg), u, ng, nd, eps);
  {
    const u128 excl = pre + woff + (inc - tsum);
    const double tj0d = (double)tj0;
    int jr = 0;
    if (k0 < nv && off + base + k0 != 0) jr = slot_rel(excl, u, ng, nd, kappa, eps, tj0d, tj0);
    u128 run = excl;
    if (P.multinomial) {   // the exact cdf per particle (filtering.py:94-95); no emission
#pragma unroll
      for (int q = 0; q < RSS_ITEMS; ++q) {
        const int k = k0 + q;
        if (k < nv) {
          run += weight(k);
          P.cdf[base + k] = (k == klast) ? 1.0 : cdf_round(run);
        }
      }
      return;
    }
#pragma unroll
    for (int q = 0; q < RSS_ITEMS; ++q) {
      const int k = k0 + q;
      int h = -1;   // no slot
      if (k < nv) {
        run += weight(k);
        const int jend = (k == klast) ? (int)(ng - tj0) : slot_rel(run, u, ng, nd, kappa, eps, tj0d, tj0);
        if (jend > jr) h = jr;
        jr = jend;
      }
      sm.hp[k] = h;
    }
  }
  // slots in chunks of RSS_TILE: heads, block max-scan, coalesced writes
  bool oob = false;
  const int m_slots = (int)(tj1 - tj0);
  int carry = -1;
  for (int c0 = 0; c0 < m_slots; c0 += RSS_TILE) {
#pragma unroll
    for (int q = 0; q < RSS_ITEMS; ++q) sm.stage[k0 + q] = -1;
    __syncthreads();
#pragma unroll
    for (int q = 0; q < RSS_ITEMS; ++q) {
      const u32 hr = (u32)(sm.hp[k0 + q] - c0);   // no head: (u32)(-1 - c0) >= 2^31
      if (hr < (u32)RSS_TILE) sm.stage[hr] = k0 + q;
    }
    __syncthreads();
    int tmax = -1;
#pragma unroll
    for (int q = 0; q < RSS_ITEMS; ++q) tmax = max(tmax, sm.stage[k0 + q]);
    int incl = tmax;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int o = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl = max(incl, o);
    }
    if (lane == 31) sm.s_wmax[wi] = incl;
    int excl_l = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) excl_l = -1;
    __syncthreads();
    int prev = carry, total = carry;
#pragma unroll
    for (int w = 0; w < SCAN_BLOCK / 32; ++w) {
      if (w < wi) prev = max(prev, sm.s_wmax[w]);
      total = max(total, sm.s_wmax[w]);
    }
    int runm = max(prev, excl_l);
#pragma unroll
    for (int q = 0; q < RSS_ITEMS; ++q) {
      runm = max(runm, sm.stage[k0 + q]);
      sm.stage[k0 + q] = runm;
    }
    __syncthreads();
    const int cm = min(RSS_TILE, m_slots - c0);
    const i64 w0 = tj0 + c0 - lo;
    const int ib = (int)base;
    for (int k = threadIdx.x; k < cm; k += SCAN_BLOCK) {
      const i64 kk = w0 + k;
      if (kk >= 0 && kk < cap) P.anc_out[kk] = ib + sm.stage[k];
      else oob = true;
    }
    carry = total;
    __syncthreads();
  }
  if (oob) set_flag(C, PCS_FLAG_CAPACITY);
  RS_PROBE(4);
}

// Multinomial resampling of the fused loops (filtering.py:96-97,100): point
// j = philox_multinomial_u(seed, frame, j) (the general path's
// pcs_philox_multinomial_points), ancestor = searchsorted(cdf, p, 'right')
// over the exact cdf the resampler wrote (N-1 at most).
__global__ void __launch_bounds__(256) k_multinomial_emit(TrackParams P) {
  TrackCtl* C = P.ctl;
  if (!C->do_resample) return;   // the resampler wrote the identity
  const u32 f = C->res_frame;
  const i64 n = P.n;
  const double* __restrict__ cdf = P.cdf;
  for (i64 j = blockIdx.x * (i64)blockDim.x + threadIdx.x; j < n; j += (i64)gridDim.x * blockDim.x) {
    const double p = philox_multinomial_u(P.seed, f, (u64)j);
    i64 lo = 0, hi = n;   // first index with cdf > p
    while (lo < hi) {
      const i64 mid = (lo + hi) >> 1;
      if (__ldg(cdf + mid) <= p) lo = mid + 1;
      else hi = mid;
    }
    P.anc_out[j] = (int)((lo < n) ? lo : n - 1);
  }
}

constexpr size_t S1_SMEM = sizeof(S1Smem);
constexpr size_t S1_SMEM_Q = sizeof(S1Smem) + sizeof(S1Queue);   // k_pc_step1<., true>

}  // namespace pcs
