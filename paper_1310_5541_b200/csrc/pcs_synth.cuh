// pcs_synth.cuh — GPU scene synthesis: ideal frames of
// one or many Gaussian spots on a constant background (synthesis.py:124-130,
// render_clean_frame) and Poisson measurement noise per pixel
// (synthesis.py:133-150, render_sequence), for the c2-c5 benchmark scenes.
//
// Ideal frame: every spot adds I0 gx gy (float64, gx = exp(-(xi - x)^2 /
// (2 s^2))) over its window of +-ceil(wr s) pixels (outside it the term is
// < I0 exp(-wr^2/2)); contributions are rounded once to 2^-32 and summed as
// unsigned 64-bit integers, so the frame does not depend on the order in
// which spots are rendered (deterministic for any spot count).
// Noise: pixel p of frame k is Poisson(lambda) drawn from the Philox stream
// (seed, p, k, 0x80000000 | iteration): sequential-search inversion for
// lambda < 10, Hörmann's transformed rejection (PTRS, 1993) above; optional
// Gaussian read noise clamped at 0 (synthesis.py:146-148).
#pragma once
#include "pcs_common.cuh"

namespace pcs {

constexpr u32 TAG_SYNTH_W = 0x80000000u;   // counter word w of the synthesis stream

// ideal-frame accumulation: one thread per (spot, window pixel)
__global__ void k_synth_spots(const double* __restrict__ spots, i64 S, i64 W, i64 H, double inv2s2,
                              int r, u64* __restrict__ acc) {
  const int side = 2 * r + 1;
  const i64 total = S * (i64)side * side;
  for (i64 g = blockIdx.x * (i64)blockDim.x + threadIdx.x; g < total; g += (i64)gridDim.x * blockDim.x) {
    const i64 s = g / ((i64)side * side);
    const int w = (int)(g % ((i64)side * side));
    const double x = spots[3 * s], y = spots[3 * s + 1], i0 = spots[3 * s + 2];
    const i64 px = (i64)floor(x) - r + (w % side), py = (i64)floor(y) - r + (w / side);
    if (px < 0 || px >= W || py < 0 || py >= H || !(i0 > 0.0)) continue;
    const double dx = (double)px - x, dy = (double)py - y;
    const double v = i0 * (exp(-(dx * dx) * inv2s2) * exp(-(dy * dy) * inv2s2));
    const u64 q = (u64)llrint(v * 4294967296.0);   // round(v 2^32), v < 2^31
    if (q) atomicAdd((unsigned long long*)(acc + py * W + px), (unsigned long long)q);
  }
}

__device__ __forceinline__ void synth_uniforms(u64 seed, u32 frame, u64 pix, u32 iter, double& u0,
                                               double& u1) {
  const u32x4 r = philox4x32_10({(u32)pix, (u32)(pix >> 32), frame, TAG_SYNTH_W | iter}, (u32)seed,
                                (u32)(seed >> 32));
  u0 = u01_double(r.x, r.y);
  u1 = u01_double(r.z, r.w);
}

// Poisson(lam) sample from the pixel's counter stream
__device__ double synth_poisson(double lam, u64 seed, u32 frame, u64 pix) {
  if (!(lam > 0.0)) return 0.0;
  double u0, u1;
  if (lam < 10.0) {   // inversion: smallest k with F(k) > u
    synth_uniforms(seed, frame, pix, 0u, u0, u1);
    double p = exp(-lam), F = p;
    int k = 0;
    while (u0 > F && k < 1000) {
      ++k;
      p *= lam / k;
      F += p;
    }
    return (double)k;
  }
  // PTRS (Hörmann 1993), two uniforms per trial
  const double slam = sqrt(lam), loglam = log(lam);
  const double b = 0.931 + 2.53 * slam;
  const double a = -0.059 + 0.02483 * b;
  const double invalpha = 1.1239 + 1.1328 / (b - 3.4);
  const double vr = 0.9277 - 3.6224 / (b - 2.0);
  for (u32 it = 0; it < (1u << 20); ++it) {
    synth_uniforms(seed, frame, pix, it, u0, u1);
    const double U = u0 - 0.5, V = u1;
    const double us = 0.5 - fabs(U);
    const double k = floor((2.0 * a / us + b) * U + lam + 0.43);
    if (us >= 0.07 && V <= vr) return k;
    if (k < 0.0 || (us < 0.013 && V > us)) continue;
    if (log(V) + log(invalpha) - log(a / (us * us) + b) <= -lam + k * loglam - lgamma(k + 1.0))
      return k;
  }
  return floor(lam);   // not reached in practice
}

// finalize: lambda = bg + acc 2^-32; noisy or ideal float32 pixel
__global__ void k_synth_finalize(const u64* __restrict__ acc, i64 npix, double bg, int noise,
                                 double read_std, u64 seed, u32 frame, float* __restrict__ out) {
  for (i64 p = blockIdx.x * (i64)blockDim.x + threadIdx.x; p < npix; p += (i64)gridDim.x * blockDim.x) {
    const double lam = bg + (double)acc[p] * 2.3283064365386963e-10;
    double v = lam;
    if (noise) {
      v = synth_poisson(lam, seed, frame, (u64)p);
      if (read_std > 0.0) {
        float z0, z1;
        const u32x4 r = philox4x32_10({(u32)p, (u32)((u64)p >> 32), frame, TAG_SYNTH_W | 0x00FFFFFFu},
                                      (u32)seed, (u32)(seed >> 32));
        box_muller(r.x, r.y, z0, z1);
        v = fmax(v + read_std * (double)z0, 0.0);
      }
    }
    out[p] = (float)v;
  }
}

}  // namespace pcs
