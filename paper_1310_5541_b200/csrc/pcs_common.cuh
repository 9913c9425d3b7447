// pcs_common.cuh — shared device helpers for the B200 pcSIR / SIR filter step.
//
// Everything here is sm_100a device code (plus a few host-callable inline
// helpers). Arithmetic conventions that the CPU oracle (oracle/) restates
// bit-for-bit are marked CANONICAL.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/pcsir_b200.h"

typedef unsigned __int128 u128;
typedef __int128 i128;
typedef unsigned long long u64;
typedef long long i64;
typedef unsigned int u32;

namespace pcs {

// ---------------------------------------------------------------------------
// Fixed-point scales (CANONICAL). Every reduction whose result feeds a
// decision (dummy means, normaliser, estimate, ESS, cumulative weights) is an
// exact integer sum of per-element values rounded once to 2^-F. Integer sums
// are order-independent, so results are deterministic, identical between the
// fused and the general path, and invariant to the number of GPUs.
// ---------------------------------------------------------------------------
constexpr int FX_STATE = 40;   // state components      (dummy sums, estimate)
constexpr int FX_WQ = 62;      // normalised weights    (estimate)
constexpr int FX_W2 = 120;     // squared weights       (ESS)
constexpr int FX_S = 95;       // exp(loglik - max)     (normaliser)
constexpr int FX_CDF = 120;    // normalised weights    (resampling cdf)

// ---------------------------------------------------------------------------
// int128 helpers
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ int clz64(u64 x) {
#ifdef __CUDA_ARCH__
  return __clzll((long long)x);
#else
  return x ? __builtin_clzll(x) : 64;
#endif
}

__host__ __device__ __forceinline__ double u64_to_f64_rn(u64 x) {
#ifdef __CUDA_ARCH__
  return __ull2double_rn(x);
#else
  return (double)x;  // x86-64: round-to-nearest-even
#endif
}

// CANONICAL: correctly rounded (nearest-even) conversion of an unsigned
// 128-bit integer to float64.
__host__ __device__ __forceinline__ double u128_to_f64_rn(u128 v) {
  u64 hi = (u64)(v >> 64);
  if (hi == 0) return u64_to_f64_rn((u64)v);
  int lz = clz64(hi);
  u128 m = v << lz;                 // top bit at position 127
  u64 t = (u64)(m >> 64);           // top 64 bits
  bool sticky = ((u64)m) != 0;
  u64 keep = t >> 11;               // 53 bits
  u64 rem = t & 0x7FFull;
  bool up = (rem > 0x400ull) || (rem == 0x400ull && (sticky || (keep & 1ull)));
  keep += up ? 1ull : 0ull;
  int e = 75 - lz;                  // value = keep * 2^e
  if (keep == (1ull << 53)) { keep >>= 1; e += 1; }
#ifdef __CUDA_ARCH__
  return scalbn((double)keep, e);
#else
  return __builtin_scalbn((double)keep, e);
#endif
}

// RN64(v) * 2^-s for v < 2^127 and a result in the normal range; same value
// as scalbn(u128_to_f64_rn(v), -s): the top 64 bits with the discarded low
// bits OR-ed into bit 0 (a sticky bit below the 11 rounding bits) round
// exactly like the full 128-bit value, and the power-of-two scale is exact.
__device__ __forceinline__ double u128_to_f64_rn_scaled(u128 v, int s) {
  u64 hi = (u64)(v >> 64), lo = (u64)v;
  if (hi == 0) return __dmul_rn(__ull2double_rn(lo), __longlong_as_double((i64)(1023 - s) << 52));
  int lz = __clzll((long long)hi);
  u64 t = lz ? ((hi << lz) | (lo >> (64 - lz))) : hi;
  u64 rest = lz ? (lo << lz) : lo;
  t |= (rest != 0ull) ? 1ull : 0ull;
  return __dmul_rn(__ull2double_rn(t), __longlong_as_double((i64)(1023 + 64 - lz - s) << 52));
}

// RN64(v) * 2^-s for a signed 128-bit v (fast path when the result is a
// normal number, scalbn otherwise); same value as scalbn(i128_to_f64_rn(v), -s)
__device__ __forceinline__ double i128_to_f64_scaled(i128 v, int s);

__host__ __device__ __forceinline__ double i128_to_f64_rn(i128 v) {
  if (v < 0) return -u128_to_f64_rn((u128)(-v));
  return u128_to_f64_rn((u128)v);
}

__device__ __forceinline__ double i128_to_f64_scaled(i128 v, int s) {
  const bool neg = v < 0;
  const u128 a = neg ? (u128)(-v) : (u128)v;
  const u64 hi = (u64)(a >> 64);
  const int lz = hi ? __clzll((long long)hi) : 64 + __clzll((long long)(u64)a);
  if (a == 0) return 0.0;
  if (1023 + 127 - lz - s <= 0) return scalbn(i128_to_f64_rn(v), -s);   // subnormal result
  const double r = u128_to_f64_rn_scaled(a, s);
  return neg ? -r : r;
}

// CANONICAL: round(m * 2^s) for a non-negative integer significand m,
// round-half-to-even when s < 0.
__host__ __device__ __forceinline__ u128 shift_round(u64 m, int s) {
  if (m == 0) return 0;
  if (s >= 0) return ((u128)m) << s;
  int r = -s;
  if (r > 64) return 0;             // m < 2^64 <= 2^(r-1): rounds to 0
  if (r == 64) return (m > (1ull << 63)) ? 1 : 0;  // tie (m == 2^63) -> even 0
  u64 q = m >> r;
  u64 rem = m & ((1ull << r) - 1ull);
  u64 half = 1ull << (r - 1);
  if (rem > half || (rem == half && (q & 1ull))) q += 1;
  return (u128)q;
}

// CANONICAL: round(v * 2^F) for a float32 value, as a signed 128-bit integer.
__host__ __device__ __forceinline__ i128 f32_to_fixed(float v, int F) {
#ifdef __CUDA_ARCH__
  u32 bits = __float_as_uint(v);
#else
  u32 bits;
  __builtin_memcpy(&bits, &v, 4);
#endif
  u32 ef = (bits >> 23) & 0xFFu;
  u64 m = bits & 0x7FFFFFu;
  int e;
  if (ef == 0) {
    e = -149;
  } else {
    m |= 0x800000u;
    e = (int)ef - 150;
  }
  i128 q = (i128)shift_round(m, e + F);
  return (bits >> 31) ? -q : q;
}

// CANONICAL: round(v * 2^F) for a float64 value (finite), signed 128-bit.
__host__ __device__ __forceinline__ i128 f64_to_fixed(double v, int F) {
#ifdef __CUDA_ARCH__
  u64 bits = (u64)__double_as_longlong(v);
#else
  u64 bits;
  __builtin_memcpy(&bits, &v, 8);
#endif
  u32 ef = (u32)((bits >> 52) & 0x7FFull);
  u64 m = bits & 0xFFFFFFFFFFFFFull;
  int e;
  if (ef == 0) {
    e = -1074;
  } else {
    m |= (1ull << 52);
    e = (int)ef - 1075;
  }
  i128 q = (i128)shift_round(m, e + F);
  return (bits >> 63) ? -q : q;
}

// Deterministic atomic add of a signed 128-bit value into two u64 words
// [lo, hi]. The final value is the exact sum mod 2^128 regardless of the
// order of the adds: every wrap of the low word contributes exactly one carry.
__device__ __forceinline__ void atomic_add_i128(u64* p, i128 v) {
  u64 vlo = (u64)v;
  u64 vhi = (u64)((u128)v >> 64);
  if (vlo) {
    u64 old = atomicAdd(p, vlo);
    if (old + vlo < old) vhi += 1ull;
  }
  if (vhi) atomicAdd(p + 1, vhi);
}

// five int128 atomic adds at p0 + c * stride (c = 0..4): the five low-word
// atomics are issued back to back (one round trip), then the high words with
// their carries
__device__ __forceinline__ void atomic_add_i128_x5(u64* p0, i64 stride, const i128 (&v)[5]) {
  u64 old[5];
#pragma unroll
  for (int c = 0; c < 5; ++c) {
    const u64 vlo = (u64)v[c];
    old[c] = vlo ? atomicAdd(p0 + c * stride, vlo) : 0ull;
  }
#pragma unroll
  for (int c = 0; c < 5; ++c) {
    const u64 vlo = (u64)v[c];
    u64 vhi = (u64)((u128)v[c] >> 64);
    if (vlo && old[c] + vlo < old[c]) vhi += 1ull;
    if (vhi) atomicAdd(p0 + c * stride + 1, vhi);
  }
}

__device__ __forceinline__ i128 load_i128(const u64* p) {
  return (i128)(((u128)p[1] << 64) | (u128)p[0]);
}

// Warp-level i128 sum (deterministic butterfly order).
__device__ __forceinline__ i128 warp_sum_i128(i128 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    u64 lo = (u64)v, hi = (u64)((u128)v >> 64);
    u64 olo = __shfl_xor_sync(0xffffffffu, lo, o);
    u64 ohi = __shfl_xor_sync(0xffffffffu, hi, o);
    v += (i128)(((u128)ohi << 64) | (u128)olo);
  }
  return v;
}

__device__ __forceinline__ u128 shfl_up_u128(u128 v, int d) {
  u64 lo = (u64)v, hi = (u64)(v >> 64);
  lo = __shfl_up_sync(0xffffffffu, lo, d);
  hi = __shfl_up_sync(0xffffffffu, hi, d);
  return ((u128)hi << 64) | (u128)lo;
}

__device__ __forceinline__ u128 shfl_u128(u128 v, int src) {
  u64 lo = (u64)v, hi = (u64)(v >> 64);
  lo = __shfl_sync(0xffffffffu, lo, src);
  hi = __shfl_sync(0xffffffffu, hi, src);
  return ((u128)hi << 64) | (u128)lo;
}

// Order-preserving float <-> int mapping for deterministic atomicMax.
__device__ __forceinline__ int float_to_ordered(float f) {
  int i = __float_as_int(f);
  return (i >= 0) ? i : (i ^ 0x7FFFFFFF);
}
__device__ __forceinline__ float ordered_to_float(int i) {
  return __int_as_float((i >= 0) ? i : (i ^ 0x7FFFFFFF));
}

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11) counter-based RNG.
// ---------------------------------------------------------------------------
struct u32x4 { u32 x, y, z, w; };

__host__ __device__ __forceinline__ void mulhilo32(u32 a, u32 b, u32& hi, u32& lo) {
#ifdef __CUDA_ARCH__
  lo = a * b;
  hi = __umulhi(a, b);
#else
  u64 p = (u64)a * (u64)b;
  lo = (u32)p;
  hi = (u32)(p >> 32);
#endif
}

__host__ __device__ __forceinline__ u32x4 philox4x32_10(u32x4 c, u32 k0, u32 k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    u32 hi0, lo0, hi1, lo1;
    mulhilo32(0xD2511F53u, c.x, hi0, lo0);
    mulhilo32(0xCD9E8D57u, c.z, hi1, lo1);
    u32x4 n;
    n.x = hi1 ^ c.y ^ k0;
    n.y = lo1;
    n.z = hi0 ^ c.w ^ k1;
    n.w = lo0;
    c = n;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// Round keys of a seed, (k0 + r W0, k1 + r W1) for r = 0..9. Kernels that
// take a PhiloxKey as a launch parameter read the keys as constant-bank
// operands of the xor (no per-thread key schedule); same stream as
// philox4x32_10(c, (u32)seed, (u32)(seed >> 32)).
struct PhiloxKey {
  u32 a[10], b[10];
};
__host__ __device__ __forceinline__ PhiloxKey philox_key(u64 seed) {
  PhiloxKey K;
  u32 k0 = (u32)seed, k1 = (u32)(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    K.a[r] = k0;
    K.b[r] = k1;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return K;
}
__device__ __forceinline__ u32x4 philox4x32_10k(u32x4 c, const PhiloxKey& K) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const u64 p0 = (u64)0xD2511F53u * c.x;   // one IMAD.WIDE.U32 each
    const u64 p1 = (u64)0xCD9E8D57u * c.z;
    u32x4 n;
    n.x = (u32)(p1 >> 32) ^ c.y ^ K.a[r];
    n.y = (u32)p1;
    n.z = (u32)(p0 >> 32) ^ c.w ^ K.b[r];
    n.w = (u32)p0;
    c = n;
  }
  return c;
}

// Stream tags (counter word w) — one per consumer so streams never overlap.
enum : u32 {
  TAG_PROPAGATE = 0x1u,
  TAG_INIT = 0x2u,
  TAG_RESAMPLE = 0x3u,
  TAG_MULTINOMIAL = 0x4u,
};

// CANONICAL uniform in (0,1) with 24 bits: ((r >> 8) + 0.5) * 2^-24 (exact in fp32)
__device__ __forceinline__ float u01_open(u32 r) {
  return ((float)(r >> 8) + 0.5f) * 5.9604644775390625e-8f;
}
// uniform in [0,1) with 24 bits (exact in fp32)
__device__ __forceinline__ float u01_closed_open(u32 r) {
  return (float)(r >> 8) * 5.9604644775390625e-8f;
}
// CANONICAL double in [0,1) from two words: (a>>5 * 2^26 + b>>6) * 2^-53
__host__ __device__ __forceinline__ double u01_double(u32 a, u32 b) {
  return ((double)(a >> 5) * 67108864.0 + (double)(b >> 6)) * (1.0 / 9007199254740992.0);
}

// Box–Muller pair in fp32 on the SFU: r = sqrt(-2 ln u1) (MUFU.LG2),
// (z0, z1) = r (cos, sin)(2 pi (u2 - 1/2)) (MUFU.SIN/COS on [-pi, pi), where
// the approximations are accurate to ~2^-21 absolute). The normals are
// defined by this function; the oracle replays them (pcs_philox_normals).
__device__ __forceinline__ void box_muller(u32 a, u32 b, float& z0, float& z1) {
  float u1 = u01_open(a);
  float u2 = u01_closed_open(b);
  float l2 = -2.0f * __logf(u1);   // >= 0 since u1 < 1 (the SFU log may round to 0 near 1)
  float r = (l2 > 0.0f) ? l2 * rsqrtf(l2) : 0.0f;   // MUFU.RSQ, not the IEEE sqrt sequence
  float s, c;
  __sincosf(6.28318530717958647692f * (u2 - 0.5f), &s, &c);
  z0 = r * c;
  z1 = r * s;
}

// Box–Muller on explicit integer uniforms: u1 = (a + 1/2) 2^-22 (a < 2^22),
// u2 = b 2^-20 (b < 2^20). Flush-to-zero SFU forms (the arguments are never
// subnormal): r = l2 * rsqrt(l2), l2 = lg2(u1) * (-2 ln 2); the angle
// 2 pi b 2^-20 - pi is one FMA.
__device__ __forceinline__ float lg2_ftz(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rsqrt_ftz(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float bm_radius22(u32 a) {
  const float u1 = fmaf((float)a, 2.384185791015625e-07f, 1.1920928955078125e-07f);
  const float l2 = lg2_ftz(u1) * -1.38629436111989061883f;   // -2 ln 2
  return (l2 > 0.0f) ? l2 * rsqrt_ftz(l2) : 0.0f;
}
__device__ __forceinline__ float bm_angle20(u32 b) {
  return fmaf((float)b, 5.9921124526782e-06f, -3.14159265358979323846f);   // 2 pi 2^-20
}

// The five standard normals used to propagate particle `idx` at `frame`
// (column order x, y, vx, vy, I0 — matches rng.normal(size=(N,5)) row
// layout in state.py:125), from ONE Philox4x32-10 block r = (x, y, z, w):
// three Box–Muller pairs on 22-bit u1 / 20-bit u2 (126 of the 128 bits):
//   pair 0: u1 = x >> 10, u2 = y >> 12           -> z0, z1
//   pair 1: u1 = z >> 10, u2 = w >> 12           -> z2, z3
//   pair 2: u1 = (x & 0x3FF) << 12 | (y & 0xFFF),
//           u2 = (z & 0x3FF) << 10 | (w >> 2 & 0x3FF) -> z4 (cosine branch)
// Exposed through pcs_philox_normals for replay; oracle/oracle.c restates it.
__device__ __forceinline__ void normals5_from_bits(const u32x4& r, float z[5]) {
  float s, c, rad;
  rad = bm_radius22(r.x >> 10);
  __sincosf(bm_angle20(r.y >> 12), &s, &c);
  z[0] = rad * c;
  z[1] = rad * s;
  rad = bm_radius22(r.z >> 10);
  __sincosf(bm_angle20(r.w >> 12), &s, &c);
  z[2] = rad * c;
  z[3] = rad * s;
  rad = bm_radius22(((r.x & 0x3FFu) << 12) | (r.y & 0xFFFu));
  z[4] = rad * __cosf(bm_angle20(((r.z & 0x3FFu) << 10) | ((r.w >> 2) & 0x3FFu)));
}
__device__ __forceinline__ void philox_normals5(u64 seed, u32 frame, u64 idx, float z[5]) {
  u32 k0 = (u32)seed, k1 = (u32)(seed >> 32);
  u32x4 r = philox4x32_10({(u32)idx, (u32)(idx >> 32), frame, (TAG_PROPAGATE << 4) | 0u}, k0, k1);
  normals5_from_bits(r, z);
}
// same normals, round keys from a launch parameter
__device__ __forceinline__ void philox_normals5k(const PhiloxKey& K, u32 frame, u64 idx, float z[5]) {
  u32x4 r = philox4x32_10k({(u32)idx, (u32)(idx >> 32), frame, (TAG_PROPAGATE << 4) | 0u}, K);
  normals5_from_bits(r, z);
}

// Two standard normals for the initial cloud (InitSpec "gauss", state.py:173)
__device__ __forceinline__ void philox_normals2_init(u64 seed, u64 idx, float z[2]) {
  u32 k0 = (u32)seed, k1 = (u32)(seed >> 32);
  u32x4 r = philox4x32_10({(u32)idx, (u32)(idx >> 32), 0u, (TAG_INIT << 4)}, k0, k1);
  box_muller(r.x, r.y, z[0], z[1]);
}

// Two uniforms in [0,1) (double) for InitSpec "uniform" (state.py:171)
__device__ __forceinline__ void philox_uniform2_init(u64 seed, u64 idx, double u[2]) {
  u32 k0 = (u32)seed, k1 = (u32)(seed >> 32);
  u32x4 r = philox4x32_10({(u32)idx, (u32)(idx >> 32), 0u, (TAG_INIT << 4) | 1u}, k0, k1);
  u[0] = u01_double(r.x, r.y);
  u[1] = u01_double(r.z, r.w);
}

// Systematic-resampling offset for `frame` (filtering.py:99 rng.random())
__host__ __device__ __forceinline__ double philox_resample_u(u64 seed, u32 frame) {
  u32x4 r = philox4x32_10({0u, 0u, frame, (TAG_RESAMPLE << 4)}, (u32)seed, (u32)(seed >> 32));
  return u01_double(r.x, r.y);
}

// Multinomial point j for `frame` (filtering.py:97 rng.random(n))
__host__ __device__ __forceinline__ double philox_multinomial_u(u64 seed, u32 frame, u64 j) {
  u32x4 r = philox4x32_10({(u32)j, (u32)(j >> 32), frame, (TAG_MULTINOMIAL << 4)}, (u32)seed,
                          (u32)(seed >> 32));
  return u01_double(r.x, r.y);
}

// ---------------------------------------------------------------------------
// Grid / cell indices (binning.py:61-67, :105) — CANONICAL, computed in
// float64 from the float32 state exactly as numpy does on the upcast value.
// ---------------------------------------------------------------------------
__device__ __forceinline__ i64 cell_axis(float p, double origin, double cell, i64 n) {
  double q = floor(__ddiv_rn(__dsub_rn((double)p, origin), cell));
  // np.clip(q, 0, n-1) then astype(int64); NaN propagates through clip and
  // astype yields INT64_MIN on x86 — map NaN to 0 and flag upstream.
  if (!(q >= 0.0)) return 0;               // negative or NaN
  double hi = (double)(n - 1);
  if (q > hi) return n - 1;
  return (i64)q;
}

struct Grid {
  double ox, oy, lx, ly;
  i64 ncols, nrows;
};

__device__ __forceinline__ void cell_of(const Grid& g, float x, float y, i64& ix, i64& iy) {
  ix = cell_axis(x, g.ox, g.lx, g.ncols);
  iy = cell_axis(y, g.oy, g.ly, g.nrows);
}

// ---------------------------------------------------------------------------
// misc
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ i64 ceil_div(i64 a, i64 b) { return (a + b - 1) / b; }

}  // namespace pcs

#define PCS_CUDA_TRY(expr)                          \
  do {                                              \
    cudaError_t _e = (expr);                        \
    if (_e != cudaSuccess) {                        \
      pcs_set_last_error(cudaGetErrorString(_e));   \
      return PCS_E_CUDA;                            \
    }                                               \
  } while (0)

void pcs_set_last_error(const char* msg);
