// pcs_weights.cuh — weight update, normalisation, estimate/ESS and the
// exact-prefix resampling scan (general path building blocks; the fused
// track reuses the device functions).
//
// Reference: filtering.py:62-72 (sis_step weight update), :75-85 (normalize),
// :88-90 (ESS), :93-100 (_resample_indices), :112-114 (posterior_mean),
// binning.py:189-194 (pcSIR broadcast).
#pragma once
#include "pcs_common.cuh"

namespace pcs {

constexpr int SCAN_BLOCK = 256;
constexpr int SCAN_ITEMS = 16;
constexpr int SCAN_TILE = SCAN_BLOCK * SCAN_ITEMS;

// ---------------------------------------------------------------------------
// block reductions (deterministic: fixed shuffle/smem tree)
// ---------------------------------------------------------------------------
template <int BLOCK>
__device__ __forceinline__ i128 block_sum_i128(i128 v, i128* sh /*[BLOCK/32]*/) {
  v = warp_sum_i128(v);
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  i128 t = 0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < BLOCK / 32; ++k) t += sh[k];
  }
  return t;  // valid in thread 0
}

// K sums with one barrier pair; results valid in thread 0
template <int BLOCK, int K>
__device__ __forceinline__ void block_sum_i128_k(i128 (&v)[K], i128* sh /*[BLOCK/32*K]*/) {
#pragma unroll
  for (int c = 0; c < K; ++c) v[c] = warp_sum_i128(v[c]);
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) {
#pragma unroll
    for (int c = 0; c < K; ++c) sh[w * K + c] = v[c];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int c = 0; c < K; ++c) {
      i128 t = 0;
      for (int q = 0; q < BLOCK / 32; ++q) t += sh[q * K + c];
      v[c] = t;
    }
  }
}

__device__ __forceinline__ double warp_max_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ordered int64 encoding of doubles for atomicMax (total order, -inf lowest)
__device__ __forceinline__ i64 f64_to_ordered(double d) {
  i64 i = __double_as_longlong(d);
  return (i >= 0) ? i : (i ^ 0x7FFFFFFFFFFFFFFFll);
}
__device__ __forceinline__ double ordered_to_f64(i64 i) {
  return __longlong_as_double((i >= 0) ? i : (i ^ 0x7FFFFFFFFFFFFFFFll));
}

// ---------------------------------------------------------------------------
// general-path scalars live in a small device struct
// ---------------------------------------------------------------------------
struct NormCtl {
  i64 max_ord;        // ordered max of logw
  u32 nonfinite;
  u32 pad;
  u64 S[2];           // sum round(exp(logw-m) * 2^FX_S)
  u64 est[5][2];      // sum Wq*V
  u64 w2[2];          // sum round(w^2 * 2^FX_W2)
};

// logw[i] = log(prior_w[i]) + ll[idx]  (float64; uniform prior drops log(1/N))
__global__ void k_weight_update(const float* __restrict__ prior_w,
                                const double* __restrict__ prior_logw,
                                const double* __restrict__ ll, const int* __restrict__ bin_of,
                                i64 n, double* __restrict__ logw) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    double l = ll[bin_of ? (i64)bin_of[i] : i];
    double p = prior_logw ? prior_logw[i] : (prior_w ? log((double)prior_w[i]) : 0.0);
    logw[i] = __dadd_rn(p, l);
  }
}

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_logw_max(const double* __restrict__ logw, i64 n,
                                                    NormCtl* ctl) {
  double m = -INFINITY;
  u32 bad = 0;
  for (i64 i = blockIdx.x * (i64)BLOCK + threadIdx.x; i < n; i += (i64)gridDim.x * BLOCK) {
    double v = logw[i];
    if (v != v || v == INFINITY) bad = 1;
    else m = fmax(m, v);
  }
  m = warp_max_f64(m);
  if ((threadIdx.x & 31) == 0) atomicMax((long long*)&ctl->max_ord, (long long)f64_to_ordered(m));
  if (bad) atomicOr(&ctl->nonfinite, 1u);
}

// CANONICAL: what = exp(logw - m) (float64); S = sum round(what * 2^95)
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_logw_sum(const double* __restrict__ logw, i64 n,
                                                    NormCtl* ctl) {
  __shared__ i128 sh[BLOCK / 32];
  double m = ordered_to_f64(ctl->max_ord);
  i128 acc = 0;
  for (i64 i = blockIdx.x * (i64)BLOCK + threadIdx.x; i < n; i += (i64)gridDim.x * BLOCK) {
    double e = exp(__dsub_rn(logw[i], m));
    acc += f64_to_fixed(e, FX_S);
  }
  i128 t = block_sum_i128<BLOCK>(acc, sh);
  if (threadIdx.x == 0) atomic_add_i128(ctl->S, t);
}

// CANONICAL: w = RN32( exp(logw - m) / RN64(S * 2^-95) )
__device__ __forceinline__ float normalised_weight(double logw, double m, double Sf) {
  return __double2float_rn(__ddiv_rn(exp(__dsub_rn(logw, m)), Sf));
}
// the same weight from a cached ex = exp(logw - m)
__device__ __forceinline__ float weight_from_ex(double ex, double Sf) {
  return __double2float_rn(__ddiv_rn(ex, Sf));
}

__global__ void k_logw_normalise(const double* __restrict__ logw, i64 n, const NormCtl* ctl,
                                 float* __restrict__ w) {
  double m = ordered_to_f64(ctl->max_ord);
  double Sf = scalbn(i128_to_f64_rn(load_i128(ctl->S)), -FX_S);
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    w[i] = normalised_weight(logw[i], m, Sf);
}

// CANONICAL estimate and ESS:
//   est_c = RN64( sum_i round(w_i 2^62) * round(s_ic 2^40) ) * 2^-102
//   ESS   = 1 / ( RN64( sum_i round(w_i^2 2^120) ) * 2^-120 )
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_estimate_ess(const float* __restrict__ s, i64 ld,
                                                        const float* __restrict__ w, i64 n,
                                                        NormCtl* ctl) {
  __shared__ i128 sh[BLOCK / 32];
  i128 acc[6] = {0, 0, 0, 0, 0, 0};
  for (i64 i = blockIdx.x * (i64)BLOCK + threadIdx.x; i < n; i += (i64)gridDim.x * BLOCK) {
    float wi = w[i];
    i128 wq = f32_to_fixed(wi, FX_WQ);
#pragma unroll
    for (int c = 0; c < 5; ++c) acc[c] += wq * f32_to_fixed(s[c * ld + i], FX_STATE);
    double w2 = (double)wi * (double)wi;  // exact
    acc[5] += f64_to_fixed(w2, FX_W2);
  }
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    i128 t = block_sum_i128<BLOCK>(acc[c], sh);
    if (threadIdx.x == 0) atomic_add_i128(c < 5 ? ctl->est[c] : ctl->w2, t);
  }
}

// ---------------------------------------------------------------------------
// Exact-prefix systematic resampling (CANONICAL)
//   W_i  = round(w_i * 2^120)                     (u128, exact for w >= 2^-97)
//   c_i  = RN64( sum_{k<=i} W_k ) * 2^-120 ;  c_{n-1} := 1.0   (filtering.py:95)
//   p_j  = RN64( RN64(u + j) / n )                              (filtering.py:99)
//   particle i owns slots j with c_{i-1} <= p_j < c_i  (searchsorted side='right',
//   filtering.py:100); slots beyond the last boundary go to particle n-1.
// ---------------------------------------------------------------------------
struct WeightSrc {
  // one of: direct fp32 weights; table lookup (pcSIR fused); loglik (SIR fused)
  const float* w;
  const u32* slot;
  const float* wtab;
  const double* ll;
  double m, Sf;
  int kind;  // 0 direct, 1 table, 2 loglik
  __device__ __forceinline__ float get(i64 i) const {
    if (kind == 0) return w[i];
    if (kind == 1) return wtab[slot[i]];
    return normalised_weight(ll[i], m, Sf);
  }
};

__device__ __noinline__ u128 cdf_fixed_slow(float w) { return (u128)f32_to_fixed(w, FX_CDF); }

__device__ __forceinline__ u128 cdf_fixed(float w) {
  // fast path (2^-97 <= w < 2^98, positive): round(w * 2^120) is an exact
  // left shift of the 24-bit significand by s = e - 30 (two 64-bit halves)
  const u32 b = __float_as_uint(w);
  const u32 ef = (b >> 23) & 0xFFu;
  if ((b >> 31) || ef < 30u) return cdf_fixed_slow(w);
  const u64 m = (u64)((b & 0x7FFFFFu) | 0x800000u);
  const int s = (int)ef - 30;
  u64 lo, hi;
  if (s < 40) {          // m << s < 2^64
    lo = m << s;
    hi = 0;
  } else if (s < 64) {
    lo = m << s;
    hi = m >> (64 - s);
  } else {
    lo = 0;
    hi = m << (s - 64);
  }
  return ((u128)hi << 64) | (u128)lo;
}

// P <= 2^121 (sum of normalised weights), so 2^-120 * RN64(P) is normal
__device__ __forceinline__ double cdf_round(u128 P) { return u128_to_f64_rn_scaled(P, FX_CDF); }

__device__ __forceinline__ double sys_point(double u, i64 j, double nd) {
  return __ddiv_rn(__dadd_rn(u, (double)j), nd);
}

// smallest j in [0, n] with p_j >= c  (p_n := +inf)
__device__ __forceinline__ i64 first_slot_at_or_above(double c, double u, i64 n) {
  double nd = (double)n;
  double g = ceil(__dsub_rn(__dmul_rn(c, nd), u));
  i64 j;
  if (!(g > 0.0)) j = 0;
  else if (g >= nd) j = n;
  else j = (i64)g;
  while (j > 0 && sys_point(u, j - 1, nd) >= c) --j;
  while (j < n && sys_point(u, j, nd) < c) ++j;
  return j;
}

// Same result as first_slot_at_or_above without a division unless
// T = c*n - u is within eps = n*2^-50 of an integer: the points satisfy
// |p_j - (u+j)/n| <= 2^-52, so away from integers J = ceil(T) exactly.
__device__ __forceinline__ i64 first_slot_fast(double c, double u, i64 n, double nd,
                                               double eps) {
  double t = fma(c, nd, -u);
  double g = ceil(t);
  double gap = g - t;
  if (gap > eps && gap < 1.0 - eps && g > 0.0 && g < nd) return (i64)g;
  return first_slot_at_or_above(c, u, n);
}

// pass 1: per-tile sums of W_i (striped, coalesced; integer sums are order-free)
__global__ void __launch_bounds__(SCAN_BLOCK) k_cdf_tiles(WeightSrc src, i64 n,
                                                          u128* __restrict__ tile_tot) {
  __shared__ i128 sh[SCAN_BLOCK / 32];
  i64 base = (i64)blockIdx.x * SCAN_TILE;
  u128 acc = 0;
#pragma unroll 4
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    i64 i = base + (i64)k * SCAN_BLOCK + threadIdx.x;
    if (i < n) acc += cdf_fixed(src.get(i));
  }
  i128 t = block_sum_i128<SCAN_BLOCK>((i128)acc, sh);
  if (threadIdx.x == 0) tile_tot[blockIdx.x] = (u128)t;
}

// pass 2: exclusive scan of tile totals (one CTA of 1024 threads)
__global__ void __launch_bounds__(1024) k_scan_tiles(const u128* __restrict__ tot, i64 ntiles,
                                                     u128* __restrict__ pre, i64* advance) {
  __shared__ u128 sh[32];
  i64 per = ceil_div(ntiles, 1024);
  i64 b0 = threadIdx.x * per, b1 = min(ntiles, b0 + per);
  u128 s = 0;
  for (i64 b = b0; b < b1; ++b) s += tot[b];
  // block exclusive scan of s
  int l = threadIdx.x & 31, w = threadIdx.x >> 5;
  u128 inc = s;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    u128 o = shfl_up_u128(inc, d);
    if (l >= d) inc += o;
  }
  if (l == 31) sh[w] = inc;
  __syncthreads();
  if (w == 0) {
    u128 v = sh[l];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      u128 o = shfl_up_u128(v, d);
      if (l >= d) v += o;
    }
    sh[l] = v;  // inclusive over warps
  }
  __syncthreads();
  u128 excl = inc - s + (w > 0 ? sh[w - 1] : (u128)0);
  for (i64 b = b0; b < b1; ++b) {
    pre[b] = excl;
    excl += tot[b];
  }
  if (advance && threadIdx.x == 0) *advance += 1;  // fused track: frame counter
}

// pass 3: blocked per-thread items, block exclusive scan, boundary slots,
// ancestor emission. mode 0: write ancestors (systematic). mode 1: write cdf.
// mode 2: identity ancestors (no resampling this frame).
__device__ __forceinline__ void cdf_emit_body(const WeightSrc& src, i64 n,
                                              const u128* __restrict__ tile_pre, double u,
                                              int* __restrict__ anc, double* __restrict__ cdf_out,
                                              int mode, float* wsh, u128* wtot) {
  i64 base = (i64)blockIdx.x * SCAN_TILE;
  if (mode == 2) {
    for (int q = 0; q < SCAN_ITEMS; ++q) {
      i64 i = base + (i64)q * SCAN_BLOCK + threadIdx.x;
      if (i < n) anc[i] = (int)i;
    }
    return;
  }
  // striped coalesced load, then blocked read from shared memory
#pragma unroll 4
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    i64 i = base + (i64)k * SCAN_BLOCK + threadIdx.x;
    wsh[k * SCAN_BLOCK + threadIdx.x] = (i < n) ? src.get(i) : 0.0f;
  }
  __syncthreads();
  u128 loc[SCAN_ITEMS];
  u128 tsum = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    tsum += cdf_fixed(wsh[threadIdx.x * SCAN_ITEMS + k]);
    loc[k] = tsum;  // thread-local inclusive
  }
  int l = threadIdx.x & 31, wi = threadIdx.x >> 5;
  u128 inc = tsum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    u128 o = shfl_up_u128(inc, d);
    if (l >= d) inc += o;
  }
  if (l == 31) wtot[wi] = inc;
  __syncthreads();
  u128 woff = 0;
  for (int k = 0; k < wi; ++k) woff += wtot[k];
  u128 excl = tile_pre[blockIdx.x] + woff + (inc - tsum);

  i64 i0 = base + (i64)threadIdx.x * SCAN_ITEMS;
  if (i0 >= n) return;
  if (mode == 0) {
    // start slot of item i0 = first slot at/above c_{i0-1}
    i64 j = (i0 == 0) ? 0 : first_slot_at_or_above(cdf_round(excl), u, n);
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
      i64 i = i0 + k;
      if (i >= n) break;
      i64 jend = (i == n - 1) ? n : first_slot_at_or_above(cdf_round(excl + loc[k]), u, n);
      for (; j < jend; ++j) anc[j] = (int)i;
    }
  } else {
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
      i64 i = i0 + k;
      if (i >= n) break;
      cdf_out[i] = (i == n - 1) ? 1.0 : cdf_round(excl + loc[k]);
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(SCAN_BLOCK) k_cdf_emit(WeightSrc src, i64 n,
                                                        const u128* __restrict__ tile_pre,
                                                        double u, int* __restrict__ anc,
                                                        double* __restrict__ cdf_out) {
  __shared__ float wsh[SCAN_TILE];
  __shared__ u128 wtot[SCAN_BLOCK / 32];
  cdf_emit_body(src, n, tile_pre, u, anc, cdf_out, MODE, wsh, wtot);
}

// multinomial: searchsorted(cdf, p_j, 'right') by binary search
__global__ void k_searchsorted(const double* __restrict__ cdf, i64 n,
                               const double* __restrict__ pts, int* __restrict__ anc) {
  for (i64 j = blockIdx.x * (i64)blockDim.x + threadIdx.x; j < n; j += (i64)gridDim.x * blockDim.x) {
    double p = pts[j];
    i64 lo = 0, hi = n;  // first index with cdf > p
    while (lo < hi) {
      i64 mid = (lo + hi) >> 1;
      if (cdf[mid] <= p) lo = mid + 1;
      else hi = mid;
    }
    anc[j] = (int)((lo < n) ? lo : n - 1);
  }
}

}  // namespace pcs
