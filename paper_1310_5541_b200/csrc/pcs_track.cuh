// pcs_track.cuh — fused per-frame filter kernels (device-resident loop).
//
// One frame of pcsir_track (binning.py:212-226) / sir_track
// (filtering.py:176-182) with ResampleConfig(threshold_fraction=1.0,
// "systematic"): propagate (+gather) -> bin -> dummies -> likelihood ->
// normalise/estimate/ESS -> exact-prefix systematic resampling. Every kernel
// reads the frame counter and all per-frame scalars from device memory, so a
// single captured CUDA graph replays any frame with no host synchronisation.
//
// Canonical arithmetic is shared with the general path (pcs_weights.cuh,
// pcs_bin.cuh): with one particle per cell the pcSIR results equal SIR
// bit-for-bit (binning.py:219 docstring, test_binning.py:182-226).
#pragma once
#include "pcs_bin.cuh"
#include "pcs_common.cuh"
#include "pcs_lik.cuh"
#include "pcs_state.cuh"
#include "pcs_weights.cuh"

namespace pcs {

constexpr i64 TABLE_CAP = 1ll << 22;   // dense bin-window cells in HBM
constexpr int MAXM = 16384;            // occupied bins handled by the fused bins kernel
constexpr int SUB_CELLS = 2048;        // shared-memory sub-window (cells)
constexpr int ACC_BLOCK = 512;
constexpr int BINS_BLOCK = 1024;

struct TrackCtl {
  // ---- per frame (reset at the end of the frame for the next one)
  i64 bbox[4];          // ix_min, ix_max, iy_min, iy_max
  i64 max_ll_ord;       // SIR: ordered-int64 max loglik (float64)
  u32 n_occ;            // pcSIR: first-touch occupied list length
  u32 wmin_bits, wmax_bits;  // SIR: min/max normalised weight (non-negative float bits)
  u64 S[2];             // SIR: normaliser
  u64 est[5][2];        // SIR: estimate numerators
  u64 w2[2];            // SIR: ESS denominator
  // ---- window of the current frame (written by the accumulate kernel)
  i64 wx0, wy0, wnx, wny;
  i64 sx0, sy0, snx, sny;
  int table_ok;
  int pad0;
  // ---- scalars consumed by the scan / emission kernels
  double m, Sf, u;
  int do_resample;
  int pad1;
  // ---- persistent
  i64 k;                // absolute frame index (since begin)
  i64 k_frames;         // frame index of frames[0]
  i64 k_out;            // frame index of out[0]
  const float* frames;
  double* out_est;
  double* out_ess;
  unsigned char* out_res;
  i64* out_occ;
  u32 flags;
  int first_bad;
  i64 evals;
  double center[2];     // previous estimate (shared-memory sub-window centre)
};

struct TrackParams {
  i64 n, ld;
  i64 H, W;
  Dyn dyn;
  Spot spot;
  Grid grid;
  u64 seed;
  u32 frame0;
  int placement;
  float* buf0;
  float* buf1;
  int* anc;
  double* ll;           // SIR: per-particle log-likelihood (float64)
  u32* pslot;           // pcSIR
  u32* tab_cnt;
  u64* tab_sum;         // [5][TABLE_CAP][2]
  float* wtab;
  u32* occ;
  TrackCtl* ctl;
};

__device__ __forceinline__ void set_flag(TrackCtl* c, u32 f) {
  atomicOr(&c->flags, f);
  atomicMin(&c->first_bad, (int)c->k);
}

__device__ __forceinline__ void reset_frame(TrackCtl* c) {
  c->bbox[0] = LLONG_MAX;
  c->bbox[1] = LLONG_MIN;
  c->bbox[2] = LLONG_MAX;
  c->bbox[3] = LLONG_MIN;
  c->max_ll_ord = LLONG_MIN;
  c->n_occ = 0;
  c->wmin_bits = 0xFFFFFFFFu;
  c->wmax_bits = 0u;
  c->S[0] = c->S[1] = 0;
  for (int q = 0; q < 5; ++q) c->est[q][0] = c->est[q][1] = 0;
  c->w2[0] = c->w2[1] = 0;
}

__device__ __forceinline__ i64 warp_min_i64(i64 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, (i64)__shfl_xor_sync(0xffffffffu, (long long)v, o));
  return v;
}
__device__ __forceinline__ i64 warp_max_i64(i64 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, (i64)__shfl_xor_sync(0xffffffffu, (long long)v, o));
  return v;
}

// ===========================================================================
// pcSIR K1: gather + propagate + bin bounding box
// ===========================================================================
__global__ void __launch_bounds__(256) k_pc_propagate(TrackParams P) {
  TrackCtl* C = P.ctl;
  if (C->flags & PCS_FLAG_CAPACITY) return;
  const i64 k = C->k;
  const float* sin = (k & 1) ? P.buf1 : P.buf0;
  float* sout = (k & 1) ? P.buf0 : P.buf1;
  i64 bx0 = LLONG_MAX, bx1 = LLONG_MIN, by0 = LLONG_MAX, by1 = LLONG_MIN;
  bool bad = false;
  const i64 n = P.n, ld = P.ld;
  for (i64 j0 = blockIdx.x * (i64)blockDim.x; j0 < n; j0 += (i64)gridDim.x * blockDim.x) {
    i64 j = j0 + threadIdx.x;
    if (j < n) {
      i64 src = (i64)__ldg(P.anc + j);
      float s[5], z[5], o[5];
#pragma unroll
      for (int c = 0; c < 5; ++c) s[c] = __ldg(sin + c * ld + src);
      philox_normals5(P.seed, P.frame0 + (u32)k, (u64)j, z);
      propagate_one(s, z, P.dyn, o);
#pragma unroll
      for (int c = 0; c < 5; ++c) sout[c * ld + j] = o[c];
      if (!(o[0] == o[0]) || !(o[1] == o[1])) bad = true;
      i64 ix, iy;
      cell_of(P.grid, o[0], o[1], ix, iy);
      bx0 = min(bx0, ix);
      bx1 = max(bx1, ix);
      by0 = min(by0, iy);
      by1 = max(by1, iy);
    }
  }
  bx0 = warp_min_i64(bx0);
  bx1 = warp_max_i64(bx1);
  by0 = warp_min_i64(by0);
  by1 = warp_max_i64(by1);
  if ((threadIdx.x & 31) == 0 && bx1 >= bx0) {
    atomicMin((long long*)&C->bbox[0], (long long)bx0);
    atomicMax((long long*)&C->bbox[1], (long long)bx1);
    atomicMin((long long*)&C->bbox[2], (long long)by0);
    atomicMax((long long*)&C->bbox[3], (long long)by1);
  }
  if (bad) set_flag(C, PCS_FLAG_NONFINITE);
}

// ===========================================================================
// pcSIR K2: per-cell exact accumulation (count + 5 sums of round(s*2^40)).
// A shared-memory sub-window around the previous estimate pre-aggregates the
// dense core (int64 deltas to a per-cell reference); everything else goes
// straight to the HBM window table. First touch of a cell appends it to the
// occupied list.
// ===========================================================================
__device__ __forceinline__ void touch_cell(const TrackParams& P, TrackCtl* C, u32 cell, u32 cnt) {
  u32 old = atomicAdd(P.tab_cnt + cell, cnt);
  if (old == 0) {
    u32 idx = atomicAdd(&C->n_occ, 1u);
    if (idx < (u32)MAXM) P.occ[idx] = cell;
  }
}

__device__ __forceinline__ i128 cell_ref(const Grid& g, int c, i64 ix, i64 iy) {
  if (c == 0) return f64_to_fixed(__dadd_rn(g.ox, __dmul_rn((double)ix, g.lx)), FX_STATE);
  if (c == 1) return f64_to_fixed(__dadd_rn(g.oy, __dmul_rn((double)iy, g.ly)), FX_STATE);
  return 0;
}

__global__ void __launch_bounds__(ACC_BLOCK) k_pc_accumulate(TrackParams P, i64 chunk) {
  TrackCtl* C = P.ctl;
  if (C->flags & PCS_FLAG_CAPACITY) return;
  extern __shared__ __align__(16) unsigned char acc_smem[];
  u32* s_cnt = (u32*)acc_smem;
  long long(*s_sum)[SUB_CELLS] = (long long(*)[SUB_CELLS])(acc_smem + SUB_CELLS * sizeof(u32));
  const i64 k = C->k;
  const float* st = (k & 1) ? P.buf0 : P.buf1;   // output of K1
  // window = bin bounding box
  const i64 wx0 = C->bbox[0], wy0 = C->bbox[2];
  const i64 wnx = C->bbox[1] - wx0 + 1, wny = C->bbox[3] - wy0 + 1;
  const double area = (double)wnx * (double)wny;
  if (!(area <= (double)TABLE_CAP)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      C->table_ok = 0;
      set_flag(C, PCS_FLAG_CAPACITY);
    }
    return;
  }
  // shared sub-window centred on the previous estimate
  i64 snx, sny;
  if (wnx * wny <= SUB_CELLS) {
    snx = wnx;
    sny = wny;
  } else if (wnx < 45) {
    snx = wnx;
    sny = SUB_CELLS / wnx;
  } else if (wny < 45) {
    sny = wny;
    snx = SUB_CELLS / wny;
  } else {
    snx = 45;
    sny = 45;
  }
  i64 cx, cy;
  cell_of(P.grid, (float)C->center[0], (float)C->center[1], cx, cy);
  i64 sx0 = min(max(cx - snx / 2, wx0), wx0 + wnx - snx);
  i64 sy0 = min(max(cy - sny / 2, wy0), wy0 + wny - sny);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    C->wx0 = wx0; C->wy0 = wy0; C->wnx = wnx; C->wny = wny;
    C->sx0 = sx0; C->sy0 = sy0; C->snx = snx; C->sny = sny;
    C->table_ok = 1;
  }
  for (int q = threadIdx.x; q < SUB_CELLS; q += ACC_BLOCK) {
    s_cnt[q] = 0;
#pragma unroll
    for (int c = 0; c < 5; ++c) s_sum[c][q] = 0;
  }
  __syncthreads();
  const i64 n = P.n, ld = P.ld;
  const i64 i_begin = (i64)blockIdx.x * chunk, i_end = min(n, i_begin + chunk);
  bool range = false;
  const i128 LIM = (i128)1 << 47;
  for (i64 i = i_begin + threadIdx.x; i < i_end; i += ACC_BLOCK) {
    float s[5];
#pragma unroll
    for (int c = 0; c < 5; ++c) s[c] = st[c * ld + i];
    i64 ix, iy;
    cell_of(P.grid, s[0], s[1], ix, iy);
    u32 cell = (u32)((iy - wy0) * wnx + (ix - wx0));
    P.pslot[i] = cell;
    i128 V[5];
#pragma unroll
    for (int c = 0; c < 5; ++c) {
      V[c] = f32_to_fixed(s[c], FX_STATE);
      if (fabsf(s[c]) >= 16777216.0f) range = true;
    }
    i64 lx = ix - sx0, ly = iy - sy0;
    bool in_sub = (lx >= 0 && lx < snx && ly >= 0 && ly < sny);
    i128 D[5];
    if (in_sub) {
#pragma unroll
      for (int c = 0; c < 5; ++c) {
        D[c] = V[c] - cell_ref(P.grid, c, ix, iy);
        if (D[c] >= LIM || D[c] <= -LIM) in_sub = false;
      }
    }
    if (in_sub) {
      int q = (int)(ly * snx + lx);
      atomicAdd(s_cnt + q, 1u);
#pragma unroll
      for (int c = 0; c < 5; ++c) atomicAdd((unsigned long long*)&s_sum[c][q], (unsigned long long)(long long)D[c]);
    } else {
      touch_cell(P, C, cell, 1u);
#pragma unroll
      for (int c = 0; c < 5; ++c) atomic_add_i128(P.tab_sum + ((i64)c * TABLE_CAP + cell) * 2, V[c]);
    }
  }
  if (range) atomicOr(&C->flags, (u32)PCS_FLAG_RANGE);
  __syncthreads();
  const int subn = (int)(snx * sny);
  for (int q = threadIdx.x; q < subn; q += ACC_BLOCK) {
    u32 cnt = s_cnt[q];
    if (!cnt) continue;
    i64 ix = sx0 + q % snx, iy = sy0 + q / snx;
    u32 cell = (u32)((iy - wy0) * wnx + (ix - wx0));
    touch_cell(P, C, cell, cnt);
#pragma unroll
    for (int c = 0; c < 5; ++c) {
      i128 tot = (i128)s_sum[c][q] + (i128)cnt * cell_ref(P.grid, c, ix, iy);
      atomic_add_i128(P.tab_sum + ((i64)c * TABLE_CAP + cell) * 2, tot);
    }
  }
}

// ===========================================================================
// pcSIR K3 (one CTA): dummies, likelihood per occupied bin, normaliser,
// per-cell weights, estimate, ESS, resampling decision. Zeroes the table
// cells it consumed so the table is clean for the next frame.
// ===========================================================================
template <int MAXS>
__global__ void __launch_bounds__(BINS_BLOCK) k_pc_bins(TrackParams P) {
  TrackCtl* C = P.ctl;
  extern __shared__ __align__(16) double s_ll[];  // [MAXM]
  __shared__ i128 s_red[BINS_BLOCK / 32];
  __shared__ long long s_max;
  __shared__ unsigned s_wmin, s_wmax;
  const int t = threadIdx.x;
  const i64 k = C->k;
  const i64 ko = k - C->k_out;
  bool capacity = (C->flags & PCS_FLAG_CAPACITY) || C->n_occ > (u32)MAXM || !C->table_ok;
  if (capacity) {
    if (t == 0) {
      set_flag(C, PCS_FLAG_CAPACITY);
      C->do_resample = 0;
      C->out_occ[ko] = -1;
      reset_frame(C);
    }
    return;
  }
  const int M = (int)C->n_occ;
  const float* frame = C->frames + (k - C->k_frames) * P.H * P.W;
  if (t == 0) {
    s_max = LLONG_MIN;
    s_wmin = 0xFFFFFFFFu;
    s_wmax = 0u;
  }
  __syncthreads();
  // 1) dummies + likelihood
  long long lmax = LLONG_MIN;
  for (int b = t; b < M; b += BINS_BLOCK) {
    u32 cell = P.occ[b];
    u32 cnt = P.tab_cnt[cell];
    float d[5];
#pragma unroll
    for (int c = 0; c < 5; ++c) {
      double num = i128_to_f64_rn(load_i128(P.tab_sum + ((i64)c * TABLE_CAP + cell) * 2));
      d[c] = __double2float_rn(scalbn(__ddiv_rn(num, (double)cnt), -FX_STATE));
    }
    if (P.placement == 1) {
      i64 ix = C->wx0 + cell % C->wnx, iy = C->wy0 + cell / C->wnx;
      d[0] = __double2float_rn(__dadd_rn(P.grid.ox, __dmul_rn((double)ix + 0.5, P.grid.lx)));
      d[1] = __double2float_rn(__dadd_rn(P.grid.oy, __dmul_rn((double)iy + 0.5, P.grid.ly)));
    }
    double ll = loglik_dispatch<MAXS>(frame, P.H, P.W, d[0], d[1], d[4], P.spot);
    s_ll[b] = ll;
    lmax = max(lmax, (long long)f64_to_ordered(ll));
  }
  atomicMax(&s_max, lmax);
  __syncthreads();
  const double m = ordered_to_f64((i64)s_max);
  const bool bad_m = !(m == m) || m == INFINITY;
  const bool degenerate = (m == -INFINITY);
  // 2) normaliser S = sum_b cnt_b * round(exp(ll_b - m) * 2^95)
  i128 acc = 0;
  for (int b = t; b < M; b += BINS_BLOCK) {
    u32 cnt = P.tab_cnt[P.occ[b]];
    acc += (i128)cnt * f64_to_fixed(exp(__dsub_rn(s_ll[b], m)), FX_S);
  }
  i128 Sfix = block_sum_i128<BINS_BLOCK>(acc, s_red);
  __shared__ double s_Sf;
  if (t == 0) s_Sf = scalbn(i128_to_f64_rn(Sfix), -FX_S);
  __syncthreads();
  const double Sf = s_Sf;
  // 3) weights per cell, estimate, ESS; zero the consumed table cells
  i128 e[6] = {0, 0, 0, 0, 0, 0};
  for (int b = t; b < M; b += BINS_BLOCK) {
    u32 cell = P.occ[b];
    u32 cnt = P.tab_cnt[cell];
    float w = normalised_weight(s_ll[b], m, Sf);
    P.wtab[cell] = w;
    atomicMin(&s_wmin, __float_as_uint(w));
    atomicMax(&s_wmax, __float_as_uint(w));
    i128 wq = f32_to_fixed(w, FX_WQ);
#pragma unroll
    for (int c = 0; c < 5; ++c) {
      u64* p = P.tab_sum + ((i64)c * TABLE_CAP + cell) * 2;
      e[c] += wq * load_i128(p);
      p[0] = 0;
      p[1] = 0;
    }
    e[5] += (i128)cnt * f64_to_fixed((double)w * (double)w, FX_W2);
    P.tab_cnt[cell] = 0;
  }
  double est[5];
  double w2f = 0;
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    i128 tot = block_sum_i128<BINS_BLOCK>(e[c], s_red);
    if (t == 0) {
      if (c < 5) est[c] = scalbn(i128_to_f64_rn(tot), -(FX_WQ + FX_STATE));
      else w2f = scalbn(i128_to_f64_rn(tot), -FX_W2);
    }
  }
  if (t == 0) {
    double ess = 1.0 / w2f;
    bool flag_bad = degenerate || bad_m;
    if (degenerate) set_flag(C, PCS_FLAG_DEGENERATE);
    if (bad_m) set_flag(C, PCS_FLAG_NONFINITE);
    for (int c = 0; c < 5; ++c) C->out_est[ko * 5 + c] = est[c];
    C->out_ess[ko] = ess;
    int res = (!flag_bad && ess < (double)P.n) ? 1 : 0;   // threshold_fraction = 1.0
    // no resampling with unequal weights -> non-uniform prior next frame:
    // only the general path carries per-particle prior weights
    if (!res && !flag_bad && s_wmin != s_wmax) set_flag(C, PCS_FLAG_CAPACITY);
    C->out_res[ko] = (unsigned char)res;
    C->out_occ[ko] = M;
    C->evals += M;
    C->do_resample = res;
    C->m = m;
    C->Sf = Sf;
    C->u = philox_resample_u(P.seed, P.frame0 + (u32)k);
    if (!flag_bad) {
      C->center[0] = est[0];
      C->center[1] = est[1];
    }
    reset_frame(C);
  }
}

// ===========================================================================
// SIR K1: gather + propagate + per-particle likelihood + max
// ===========================================================================
template <int MAXS>
__global__ void __launch_bounds__(256) k_sir_propagate_lik(TrackParams P) {
  TrackCtl* C = P.ctl;
  const i64 k = C->k;
  const float* sin = (k & 1) ? P.buf1 : P.buf0;
  float* sout = (k & 1) ? P.buf0 : P.buf1;
  const float* frame = C->frames + (k - C->k_frames) * P.H * P.W;
  long long lmax = LLONG_MIN;
  bool bad = false;
  const i64 n = P.n, ld = P.ld;
  for (i64 j = blockIdx.x * (i64)blockDim.x + threadIdx.x; j < n; j += (i64)gridDim.x * blockDim.x) {
    i64 src = (i64)__ldg(P.anc + j);
    float s[5], z[5], o[5];
#pragma unroll
    for (int c = 0; c < 5; ++c) s[c] = __ldg(sin + c * ld + src);
    philox_normals5(P.seed, P.frame0 + (u32)k, (u64)j, z);
    propagate_one(s, z, P.dyn, o);
#pragma unroll
    for (int c = 0; c < 5; ++c) sout[c * ld + j] = o[c];
    double ll = loglik_dispatch<MAXS>(frame, P.H, P.W, o[0], o[1], o[4], P.spot);
    P.ll[j] = ll;
    if (!(ll == ll) || ll == INFINITY) bad = true;
    lmax = max(lmax, (long long)f64_to_ordered(ll));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lmax = max(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
  if ((threadIdx.x & 31) == 0) atomicMax((long long*)&C->max_ll_ord, lmax);
  if (bad) set_flag(C, PCS_FLAG_NONFINITE);
}

// SIR K2: S = sum round(exp(ll - m) * 2^95)
__global__ void __launch_bounds__(256) k_sir_sum(TrackParams P) {
  __shared__ i128 sh[8];
  TrackCtl* C = P.ctl;
  const double m = ordered_to_f64(C->max_ll_ord);
  i128 acc = 0;
  for (i64 j = blockIdx.x * (i64)blockDim.x + threadIdx.x; j < P.n; j += (i64)gridDim.x * blockDim.x)
    acc += f64_to_fixed(exp(__dsub_rn(P.ll[j], m)), FX_S);
  i128 t = block_sum_i128<256>(acc, sh);
  if (threadIdx.x == 0) atomic_add_i128(C->S, t);
}

// SIR K3: cdf tile totals + estimate/ESS numerators in one pass
__global__ void __launch_bounds__(SCAN_BLOCK) k_sir_tiles_stats(TrackParams P,
                                                                u128* __restrict__ tile_tot) {
  __shared__ i128 sh[SCAN_BLOCK / 32];
  TrackCtl* C = P.ctl;
  const i64 k = C->k;
  const float* st = (k & 1) ? P.buf0 : P.buf1;
  const double m = ordered_to_f64(C->max_ll_ord);
  const double Sf = scalbn(i128_to_f64_rn(load_i128(C->S)), -FX_S);
  const i64 n = P.n, ld = P.ld;
  i64 base = (i64)blockIdx.x * SCAN_TILE;
  u128 acc = 0;
  i128 e[6] = {0, 0, 0, 0, 0, 0};
  bool range = false;
  unsigned wmin = 0xFFFFFFFFu, wmax = 0u;
  for (int q = 0; q < SCAN_ITEMS; ++q) {
    i64 i = base + (i64)q * SCAN_BLOCK + threadIdx.x;
    if (i < n) {
      float w = normalised_weight(P.ll[i], m, Sf);
      wmin = min(wmin, __float_as_uint(w));
      wmax = max(wmax, __float_as_uint(w));
      acc += cdf_fixed(w);
      i128 wq = f32_to_fixed(w, FX_WQ);
#pragma unroll
      for (int c = 0; c < 5; ++c) {
        float v = st[c * ld + i];
        if (fabsf(v) >= 16777216.0f) range = true;
        e[c] += wq * f32_to_fixed(v, FX_STATE);
      }
      e[5] += f64_to_fixed((double)w * (double)w, FX_W2);
    }
  }
  i128 t = block_sum_i128<SCAN_BLOCK>((i128)acc, sh);
  if (threadIdx.x == 0) tile_tot[blockIdx.x] = (u128)t;
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    i128 tt = block_sum_i128<SCAN_BLOCK>(e[c], sh);
    if (threadIdx.x == 0) atomic_add_i128(c < 5 ? C->est[c] : C->w2, tt);
  }
  if (range) atomicOr(&C->flags, (u32)PCS_FLAG_RANGE);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    wmin = min(wmin, __shfl_xor_sync(0xffffffffu, wmin, o));
    wmax = max(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&C->wmin_bits, wmin);
    atomicMax(&C->wmax_bits, wmax);
  }
}

// SIR K4 (one thread): frame outputs and resampling decision
__global__ void k_sir_finalize(TrackParams P) {
  TrackCtl* C = P.ctl;
  const i64 k = C->k, ko = k - C->k_out;
  const double mf = ordered_to_f64(C->max_ll_ord);
  const bool degenerate = (mf == -INFINITY);
  const bool bad_m = !(mf == mf) || mf == INFINITY;
  double est[5];
  for (int c = 0; c < 5; ++c) {
    est[c] = scalbn(i128_to_f64_rn(load_i128(C->est[c])), -(FX_WQ + FX_STATE));
    C->out_est[ko * 5 + c] = est[c];
  }
  double ess = 1.0 / scalbn(i128_to_f64_rn(load_i128(C->w2)), -FX_W2);
  C->out_ess[ko] = ess;
  bool flag_bad = degenerate || bad_m;
  if (degenerate) set_flag(C, PCS_FLAG_DEGENERATE);
  if (bad_m) set_flag(C, PCS_FLAG_NONFINITE);
  int res = (!flag_bad && ess < (double)P.n) ? 1 : 0;
  if (!res && !flag_bad && C->wmin_bits != C->wmax_bits) set_flag(C, PCS_FLAG_CAPACITY);
  C->out_res[ko] = (unsigned char)res;
  C->out_occ[ko] = P.n;
  C->evals += P.n;
  C->do_resample = res;
  C->m = mf;
  C->Sf = scalbn(i128_to_f64_rn(load_i128(C->S)), -FX_S);
  C->u = philox_resample_u(P.seed, P.frame0 + (u32)k);
  reset_frame(C);
}

// frame counter advance (after the tile scan, before emission)
__global__ void k_advance(TrackCtl* C) { C->k += 1; }

// emission wrapper reading the per-frame scalars from the control block
template <int KIND>
__global__ void __launch_bounds__(SCAN_BLOCK) k_track_tiles(TrackParams P, u128* __restrict__ tile_tot) {
  // KIND 1: pcSIR table lookup (SIR computes its tiles in k_sir_tiles_stats)
  __shared__ i128 sh[SCAN_BLOCK / 32];
  i64 base = (i64)blockIdx.x * SCAN_TILE;
  u128 acc = 0;
#pragma unroll 4
  for (int q = 0; q < SCAN_ITEMS; ++q) {
    i64 i = base + (i64)q * SCAN_BLOCK + threadIdx.x;
    if (i < P.n) acc += cdf_fixed(P.wtab[P.pslot[i]]);
  }
  i128 t = block_sum_i128<SCAN_BLOCK>((i128)acc, sh);
  if (threadIdx.x == 0) tile_tot[blockIdx.x] = (u128)t;
}

template <int KIND>
__global__ void __launch_bounds__(SCAN_BLOCK) k_track_emit(TrackParams P, const u128* __restrict__ tile_pre) {
  __shared__ float wsh[SCAN_TILE];
  __shared__ u128 wtot[SCAN_BLOCK / 32];
  const TrackCtl* C = P.ctl;
  WeightSrc src;
  src.w = nullptr;
  src.slot = P.pslot;
  src.wtab = P.wtab;
  src.ll = P.ll;
  src.m = C->m;
  src.Sf = C->Sf;
  src.kind = KIND;
  cdf_emit_body(src, P.n, tile_pre, C->u, P.anc, nullptr, C->do_resample ? 0 : 2, wsh, wtot);
}

constexpr size_t ACC_SMEM = SUB_CELLS * (sizeof(u32) + 5 * sizeof(long long));
constexpr size_t BINS_SMEM = MAXM * sizeof(double);

}  // namespace pcs
