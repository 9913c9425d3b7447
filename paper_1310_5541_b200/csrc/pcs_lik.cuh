// pcs_lik.cuh — spot likelihoods.
//
// Reference: _speedups.pyx:17-85 and kernels.py:24-40 (windowed Gaussian
// SSD), imaging.py:125-137 (exp(-ssd/(2 sigma_xi^2))). Window convention:
// centre pixel floor(p + 0.5), each bound clamped to the frame independently
// (_speedups.pyx:47-68) so far-out states see a border strip, never an error.
//
// Precision contract: per-pixel prediction in float32, each
// squared residual r*r added EXACTLY into a float64 accumulator (r is float32,
// so r*r is exact in float64) in row-major window order, log-likelihood
// returned in float64. Pixels come through a PixView: the frame in HBM or a
// staged shared-memory tile of it — same values, same arithmetic, same order,
// so both sources give bit-identical results.
#pragma once
#include "pcs_common.cuh"

namespace pcs {

struct Spot {
  float sigma_psf;
  float bg;
  float inv2s2;        // 1 / (2 sigma_psf^2)
  double inv_2sxi2;    // 1 / (2 sigma_xi^2)
  int hw;
  int model;           // 0 gauss-ssd, 1 erf-poisson, 2 midpoint4x4-poisson
  float erf_scale;     // sigma*sqrt(pi/2)  (model 1)
  float inv_sqrt2s;    // 1/(sqrt(2) sigma) (model 1)
  int f64;             // Poisson models: 1 = the float64 form (pcSIR cells)
  double sigma64, bg64, inv2s2_64, erf_scale64, inv_sqrt2s64;   // float64 parameters
};

// frame (H x W) view; pixel (x, y) lives at base[(y - y0) * pitch + (x - x0)]
struct PixView {
  const float* base;
  i64 pitch;
  int x0, y0;
  i64 H, W;
  __device__ __forceinline__ const float* row(int y, int x) const {
    return base + (i64)(y - y0) * pitch + (x - x0);
  }
};

__device__ __forceinline__ PixView frame_view(const float* pix, i64 H, i64 W) {
  PixView v;
  v.base = pix;
  v.pitch = W;
  v.x0 = 0;
  v.y0 = 0;
  v.H = H;
  v.W = W;
  return v;
}

__device__ __forceinline__ void window_axis(double p, int hw, i64 extent, int& lo, int& hi) {
  // cx = floor(p + 0.5); lo = clamp(cx - hw, 0, extent-1); hi = clamp(cx + hw, 0, extent-1)
  double c = floor(p + 0.5);
  double e1 = (double)(extent - 1);
  double l = c - (double)hw, h = c + (double)hw;
  l = (l < 0.0) ? 0.0 : ((l > e1) ? e1 : l);
  h = (h < 0.0) ? 0.0 : ((h > e1) ? e1 : h);
  lo = (int)l;
  hi = (int)h;
}

// float32 forms for float32 positions (bit-identical to the float64 forms):
// * pixel offset RN32(i - p), |i| < 2^24: the float64 difference is exact and
//   IEEE float subtraction is correctly rounded, so this equals
//   __double2float_rn(double(i) - double(p));
// * window_axis: for |p| < 2^23, p + 0.5f is exact unless it crosses into the
//   next binade, where the rounding cannot cross an integer, so
//   floorf(p + 0.5f) == floor((double)p + 0.5); other p use the float64 form.
__device__ __forceinline__ float pix_off(int i, float p) { return __fsub_rn((float)i, p); }

__device__ __forceinline__ void window_axis_f(float p, int hw, i64 extent, int& lo, int& hi) {
  if (fabsf(p) < 8388608.0f) {
    const int c = (int)floorf(__fadd_rn(p, 0.5f));
    const int e1 = (int)(extent - 1);
    lo = min(max(c - hw, 0), e1);
    hi = min(max(c + hw, 0), e1);
  } else {
    window_axis((double)p, hw, extent, lo, hi);
  }
}

__device__ __forceinline__ double nan_ll() { return __longlong_as_double(0x7ff8000000000000ll); }

// ---- Gaussian windowed SSD (CANONICAL hot-path arithmetic) ----------------
//   gx[i] = expf(-(d*d) * inv2s2), d = RN32(xi - x)        (fp32)
//   pred  = fmaf(I0*gx[i], gy[j], bg); r = p - pred         (fp32)
//   row_j = sum_i fma((double)r, (double)r, row_j)          (fp64, exact terms,
//                                                            column order)
//   ssd   = sum_j row_j                                     (fp64, row order)
//   ll    = -ssd * inv_2sxi2                                (fp64)
// The per-row partials let a warp evaluate one window with one lane per row
// (k_pc_bins) and still match the per-thread loop bit for bit.
template <int MAXS, bool FULL>
__device__ __forceinline__ double loglik_gauss_k(const PixView& pv, float x, float y, float i0,
                                                 const Spot& sp, int xlo, int nx, int ylo, int ny) {
  float ag[MAXS];
#pragma unroll
  for (int i = 0; i < MAXS; ++i) {
    if (FULL || i < nx) {
      float d = pix_off(xlo + i, x);
      ag[i] = i0 * expf(-(d * d) * sp.inv2s2);
    }
  }
  double ssd = 0.0;
  for (int j = 0; j < ny; ++j) {
    const float* row = pv.row(ylo + j, xlo);
    float d = pix_off(ylo + j, y);
    float gy = expf(-(d * d) * sp.inv2s2);
    float pr[MAXS];
#pragma unroll
    for (int i = 0; i < MAXS; ++i)
      if (FULL || i < nx) pr[i] = row[i];
    double racc = 0.0;
#pragma unroll
    for (int i = 0; i < MAXS; ++i) {
      if (FULL || i < nx) {
        float r = pr[i] - fmaf(ag[i], gy, sp.bg);
        racc = fma((double)r, (double)r, racc);
      }
    }
    ssd += racc;
  }
  return -ssd * sp.inv_2sxi2;
}

template <int MAXS>
__device__ __forceinline__ double loglik_gauss(const PixView& pv, float x, float y, float i0,
                                               const Spot& sp) {
  if (!(x == x) || !(y == y) || !(i0 == i0)) return nan_ll();
  int xlo, xhi, ylo, yhi;
  window_axis_f(x, sp.hw, pv.W, xlo, xhi);
  window_axis_f(y, sp.hw, pv.H, ylo, yhi);
  const int nx = xhi - xlo + 1, ny = yhi - ylo + 1;
  if (nx == MAXS) return loglik_gauss_k<MAXS, true>(pv, x, y, i0, sp, xlo, nx, ylo, ny);
  return loglik_gauss_k<MAXS, false>(pv, x, y, i0, sp, xlo, nx, ylo, ny);
}

// ---- Poisson log-likelihood ratio vs background (config 3, new) -------------
//   lambda = bg + I0 Ex(xi) Ey(yi);   ll = sum_window [ z log1p(mu/bg) - mu ],
//   mu = I0 Ex Ey. Equals the full-frame Poisson log-likelihood minus a
//   per-frame constant (pixels outside the window have lambda = bg), with
//   the lgamma(z+1) term dropped.
// model 1: Ex = integral of exp(-(t-x)^2/2s^2) over the pixel (erf form). The
//   4x4 sub-pixel supersampled integral telescopes exactly to this, so only
//   the S+1 pixel-EDGE values are evaluated: edge e_i = RN32(RN32(i - 1/2) - x),
//   C_i = erfc(|e_i| / (sqrt2 s)), and the pixel between edges a < b is
//   erfc(a) - erfc(b) (a >= 0), erfc(-b) - erfc(-a) (b <= 0), 2 - C_a - C_b
//   (straddling) times s sqrt(pi/2) — accurate in both tails, one erfc per edge.
// model 2: Ex = 1/4 sum_s exp(-((xi - 3/8 + s/4) - x)^2 / 2s^2) (mid-point 4x4).
// Per pixel the term z log1p(t) - t bg (t = mu/bg) is float32 with the
// log1p_pos below; a row is summed in float32 in column order and the rows
// in float64 in row order (every evaluation form below follows this order,
// so they agree bit for bit).
__device__ __forceinline__ float edge_off(int i, float p) {
  return __fsub_rn(__fsub_rn((float)i, 0.5f), p);   // (float)i - 1/2 exact for |i| < 2^23
}
__device__ __forceinline__ float edge_c(float e, const Spot& sp) {
  return erfcf(fabsf(e) * sp.inv_sqrt2s);
}
__device__ __forceinline__ float erf_pixel(float a, float b, float ca, float cb, const Spot& sp) {
  float d;
  if (a >= 0.0f) d = ca - cb;
  else if (b <= 0.0f) d = cb - ca;
  else d = (2.0f - ca) - cb;
  return sp.erf_scale * d;
}

__device__ __forceinline__ float psf_axis(float d, const Spot& sp) {   // model 2
  float t0 = d - 0.375f, t1 = d - 0.125f, t2 = d + 0.125f, t3 = d + 0.375f;
  return 0.25f * (expf(-(t0 * t0) * sp.inv2s2) + expf(-(t1 * t1) * sp.inv2s2) +
                  expf(-(t2 * t2) * sp.inv2s2) + expf(-(t3 * t3) * sp.inv2s2));
}
// PSF factor of pixel i along one axis (position p)
__device__ __forceinline__ float psf_pixel(int i, float p, const Spot& sp) {
  if (sp.model == 1) {
    const float a = edge_off(i, p), b = edge_off(i + 1, p);
    return erf_pixel(a, b, edge_c(a, sp), edge_c(b, sp), sp);
  }
  return psf_axis(pix_off(i, p), sp);
}

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// log1p(t) for 0 <= t < 1e30, within ~2 ulp: u = RN(1 + t) = m 2^e (m in
// [sqrt(1/2), sqrt(2))), log m = 2 atanh(s), s = (m - 1)/(m + 1) (series to
// s^9), plus the rounding error of 1 + t, (t - (u - 1))/u.
__device__ __forceinline__ float log1p_pos(float t) {
  const float u = 1.0f + t;
  const int ib = __float_as_int(u);
  const int e = (ib - 0x3f3504f3) >> 23;
  const float f = __int_as_float(ib - (e << 23)) - 1.0f;           // exact
  const float s = f * rcp_approx(2.0f + f);
  const float z = s * s;
  float q = fmaf(z, 0.22222222f, 0.28571429f);                     // 2/9, 2/7
  q = fmaf(q, z, 0.4f);
  q = fmaf(q, z, 0.66666669f);
  q = fmaf(q, z, 2.0f);
  const float ef = __int_as_float(0x4B400000 + e) - 12582912.0f;   // (float)e
  const float lu = fmaf(ef, 0.693145751953125f, fmaf(ef, 1.42860677e-06f, s * q));
  return fmaf(t - (u - 1.0f), rcp_approx(u), lu);
}

// FAST: every t = mu/bg of the window is in [0, 1e30) (checked once per
// evaluation by poisson_fast_ok); otherwise the library log1pf.
template <bool FAST>
__device__ __forceinline__ float poisson_term(float z, float t, float bg) {
  return fmaf(z, FAST ? log1p_pos(t) : log1pf(t), -t * bg);
}
__device__ __forceinline__ bool poisson_fast_ok(float i0, const Spot& sp) {
  // mu/bg <= I0 / bg * max(Ex) max(Ey); max Ex <= 2 s sqrt(pi/2) (model 1), <= 1 (model 2)
  const float pm = (sp.model == 1) ? 2.0f * sp.erf_scale : 1.0f;
  return i0 >= 0.0f && (i0 / sp.bg) * pm * pm < 1.0e30f;
}

// FULL: the window has all MAXS columns (not clamped at the frame edge), so
// the unrolled column loops carry no per-pixel guard
template <int MAXS, bool FAST, bool FULL>
__device__ __forceinline__ double loglik_poisson_k(const PixView& pv, float x, float y, float i0,
                                                   const Spot& sp, int xlo, int nx, int ylo,
                                                   int ny) {
  float ex[MAXS];
  const float inv_bg = 1.0f / sp.bg;
  if (sp.model == 1) {
    float a = edge_off(xlo, x), ca = edge_c(a, sp);
#pragma unroll
    for (int i = 0; i < MAXS; ++i) {
      if (FULL || i < nx) {
        const float b = edge_off(xlo + i + 1, x), cb = edge_c(b, sp);
        ex[i] = i0 * erf_pixel(a, b, ca, cb, sp) * inv_bg;   // mu/bg along x (times Ey later)
        a = b;
        ca = cb;
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < MAXS; ++i)
      if (FULL || i < nx) ex[i] = i0 * psf_axis(pix_off(xlo + i, x), sp) * inv_bg;
  }
  double ll = 0.0;
  float ya = edge_off(ylo, y), yca = (sp.model == 1) ? edge_c(ya, sp) : 0.0f;
  for (int j = 0; j < ny; ++j) {
    const float* row = pv.row(ylo + j, xlo);
    float ey;
    if (sp.model == 1) {
      const float yb = edge_off(ylo + j + 1, y), ycb = edge_c(yb, sp);
      ey = erf_pixel(ya, yb, yca, ycb, sp);
      ya = yb;
      yca = ycb;
    } else {
      ey = psf_axis(pix_off(ylo + j, y), sp);
    }
    float racc = 0.0f;
#pragma unroll
    for (int i = 0; i < MAXS; ++i)
      if (FULL || i < nx) racc += poisson_term<FAST>(row[i], ex[i] * ey, sp.bg);
    ll += (double)racc;
  }
  return ll;
}

template <int MAXS>
__device__ __forceinline__ double loglik_poisson(const PixView& pv, float x, float y, float i0,
                                                 const Spot& sp) {
  if (!(x == x) || !(y == y) || !(i0 == i0)) return nan_ll();
  int xlo, xhi, ylo, yhi;
  window_axis_f(x, sp.hw, pv.W, xlo, xhi);
  window_axis_f(y, sp.hw, pv.H, ylo, yhi);
  const int nx = xhi - xlo + 1, ny = yhi - ylo + 1;
  if (!poisson_fast_ok(i0, sp)) return loglik_poisson_k<MAXS, false, false>(pv, x, y, i0, sp, xlo, nx, ylo, ny);
  if (nx == MAXS) return loglik_poisson_k<MAXS, true, true>(pv, x, y, i0, sp, xlo, nx, ylo, ny);
  return loglik_poisson_k<MAXS, true, false>(pv, x, y, i0, sp, xlo, nx, ylo, ny);
}

// ---- float64 Poisson form (pcSIR cell likelihoods, any window) -------------
// The same model and window as above evaluated entirely in float64 (the
// dummies are float32, exact in float64): edge values C = erfc(|e| / (sqrt2
// s)) with e = (i - 1/2) - x, pixel integrals by the same sign cases, t =
// (I0 Ex / bg) Ey, term = z log1p(t) - t bg; a row is summed in column order
// and the rows in row order. Agrees with the float64 sub-pixel oracle to
// ~1e-12, i.e. |d log L| <= 1e-5 holds with a wide margin (R19; the
// per-particle SIR form above trades that for float32 pixel terms).
__device__ __forceinline__ double edge_c64(double e, const Spot& sp) {
  return erfc(fabs(e) * sp.inv_sqrt2s64);
}
__device__ __forceinline__ double erf_pixel64(double a, double b, double ca, double cb, const Spot& sp) {
  double d;
  if (a >= 0.0) d = ca - cb;
  else if (b <= 0.0) d = cb - ca;
  else d = (2.0 - ca) - cb;
  return sp.erf_scale64 * d;
}
__device__ __forceinline__ double psf_axis64(double d, const Spot& sp) {   // model 2
  const double t0 = d - 0.375, t1 = d - 0.125, t2 = d + 0.125, t3 = d + 0.375;
  return 0.25 * (((exp(-(t0 * t0) * sp.inv2s2_64) + exp(-(t1 * t1) * sp.inv2s2_64)) +
                  exp(-(t2 * t2) * sp.inv2s2_64)) + exp(-(t3 * t3) * sp.inv2s2_64));
}
// PSF factor of pixel i along one axis (position p), float64
__device__ __forceinline__ double psf_pixel64(int i, double p, const Spot& sp) {
  if (sp.model == 1) {
    const double a = ((double)i - 0.5) - p, b = ((double)i + 0.5) - p;
    return erf_pixel64(a, b, edge_c64(a, sp), edge_c64(b, sp), sp);
  }
  return psf_axis64((double)i - p, sp);
}
__device__ __forceinline__ double poisson_term64(double z, double t, double bg) {
  return z * log1p(t) - t * bg;
}
__device__ __forceinline__ double loglik_poisson64_generic(const PixView& pv, float x, float y,
                                                           float i0, const Spot& sp) {
  if (!(x == x) || !(y == y) || !(i0 == i0)) return nan_ll();
  int xlo, xhi, ylo, yhi;
  window_axis_f(x, sp.hw, pv.W, xlo, xhi);
  window_axis_f(y, sp.hw, pv.H, ylo, yhi);
  const double a0 = (double)i0 / sp.bg64;
  double ll = 0.0;
  for (int yy = ylo; yy <= yhi; ++yy) {
    const double ey = psf_pixel64(yy, (double)y, sp);
    const float* row = pv.row(yy, xlo);
    double racc = 0.0;
    for (int xx = xlo; xx <= xhi; ++xx) {
      const double ex = a0 * psf_pixel64(xx, (double)x, sp);
      racc += poisson_term64((double)row[xx - xlo], ex * ey, sp.bg64);
    }
    ll += racc;
  }
  return ll;
}

// F64OK: the float64 Poisson form may be requested (sp.f64); the per-particle
// SIR kernel instantiates without it (its code would cost registers there)
template <int MAXS, bool F64OK = true>
__device__ __forceinline__ double loglik_any(const PixView& pv, float x, float y, float i0,
                                             const Spot& sp) {
  if (sp.model == 0) return loglik_gauss<MAXS>(pv, x, y, i0, sp);
  if (F64OK && sp.f64) return loglik_poisson64_generic(pv, x, y, i0, sp);
  return loglik_poisson<MAXS>(pv, x, y, i0, sp);
}

// Generic window (any halfwidth): gx/gy recomputed per pixel; the per-pixel
// expressions and the accumulation order are identical to the MAXS forms, so
// results are bit-identical for any window size.
__device__ __forceinline__ double loglik_gauss_generic(const PixView& pv, float x, float y,
                                                       float i0, const Spot& sp) {
  if (!(x == x) || !(y == y) || !(i0 == i0)) return nan_ll();
  int xlo, xhi, ylo, yhi;
  window_axis_f(x, sp.hw, pv.W, xlo, xhi);
  window_axis_f(y, sp.hw, pv.H, ylo, yhi);
  double ssd = 0.0;
  for (int yy = ylo; yy <= yhi; ++yy) {
    float d = pix_off(yy, y);
    float gy = expf(-(d * d) * sp.inv2s2);
    const float* row = pv.row(yy, xlo);
    double racc = 0.0;
    for (int xx = xlo; xx <= xhi; ++xx) {
      float dx = pix_off(xx, x);
      float ag = i0 * expf(-(dx * dx) * sp.inv2s2);
      float r = row[xx - xlo] - fmaf(ag, gy, sp.bg);
      racc = fma((double)r, (double)r, racc);
    }
    ssd += racc;
  }
  return -ssd * sp.inv_2sxi2;
}

__device__ __forceinline__ double loglik_poisson_generic(const PixView& pv, float x, float y,
                                                         float i0, const Spot& sp) {
  if (!(x == x) || !(y == y) || !(i0 == i0)) return nan_ll();
  int xlo, xhi, ylo, yhi;
  window_axis_f(x, sp.hw, pv.W, xlo, xhi);
  window_axis_f(y, sp.hw, pv.H, ylo, yhi);
  const float inv_bg = 1.0f / sp.bg;
  const bool fast = poisson_fast_ok(i0, sp);
  double ll = 0.0;
  for (int yy = ylo; yy <= yhi; ++yy) {
    float ey = psf_pixel(yy, y, sp);
    const float* row = pv.row(yy, xlo);
    float racc = 0.0f;
    for (int xx = xlo; xx <= xhi; ++xx) {
      float exi = i0 * psf_pixel(xx, x, sp) * inv_bg;
      racc += fast ? poisson_term<true>(row[xx - xlo], exi * ey, sp.bg)
                   : poisson_term<false>(row[xx - xlo], exi * ey, sp.bg);
    }
    ll += (double)racc;
  }
  return ll;
}

__device__ __forceinline__ double loglik_generic(const PixView& pv, float x, float y, float i0,
                                                 const Spot& sp) {
  if (sp.model != 0 && sp.f64) return loglik_poisson64_generic(pv, x, y, i0, sp);
  return (sp.model == 0) ? loglik_gauss_generic(pv, x, y, i0, sp)
                         : loglik_poisson_generic(pv, x, y, i0, sp);
}

// dispatch: MAXS > 0 -> register-resident window, MAXS == 0 -> generic
template <int MAXS, bool F64OK = true>
__device__ __forceinline__ double loglik_dispatch(const PixView& pv, float x, float y, float i0,
                                                  const Spot& sp) {
  if constexpr (MAXS > 0) return loglik_any<MAXS, F64OK>(pv, x, y, i0, sp);
  else return loglik_generic(pv, x, y, i0, sp);
}

// Warp-cooperative evaluation of one window: lane i owns column factor i,
// lane j owns row j; row sums are accumulated in the same column order and
// added in the same row order as the per-thread loops above, so the result is
// bit-identical. All lanes return the value. Windows wider than 32 fall back
// to the per-thread generic loop on every lane.
__device__ __forceinline__ double loglik_warp(const PixView& pv, float x, float y, float i0,
                                              const Spot& sp, int lane) {
  if (!(x == x) || !(y == y) || !(i0 == i0)) return nan_ll();
  int xlo, xhi, ylo, yhi;
  window_axis_f(x, sp.hw, pv.W, xlo, xhi);
  window_axis_f(y, sp.hw, pv.H, ylo, yhi);
  const int nx = xhi - xlo + 1, ny = yhi - ylo + 1;
  if (nx > 32 || ny > 32) return loglik_generic(pv, x, y, i0, sp);
  const bool gauss = (sp.model == 0);
  const float inv_bg = 1.0f / sp.bg;
  const bool fast = !gauss && poisson_fast_ok(i0, sp);
  float colf = 0.0f, rowf = 0.0f;
  if (lane < nx) {
    float d = pix_off(xlo + lane, x);
    colf = gauss ? i0 * expf(-(d * d) * sp.inv2s2) : i0 * psf_pixel(xlo + lane, x, sp) * inv_bg;
  }
  if (lane < ny) {
    float d = pix_off(ylo + lane, y);
    rowf = gauss ? expf(-(d * d) * sp.inv2s2) : psf_pixel(ylo + lane, y, sp);
  }
  const float* row = pv.row(ylo + min(lane, ny - 1), xlo);
  double racc = 0.0;
  float racc_f = 0.0f;
  for (int i = 0; i < nx; ++i) {
    float ci = __shfl_sync(0xffffffffu, colf, i);
    if (lane < ny) {
      if (gauss) {
        float r = row[i] - fmaf(ci, rowf, sp.bg);
        racc = fma((double)r, (double)r, racc);
      } else {
        racc_f += fast ? poisson_term<true>(row[i], ci * rowf, sp.bg)
                       : poisson_term<false>(row[i], ci * rowf, sp.bg);
      }
    }
  }
  if (!gauss) racc = (double)racc_f;
  double tot = 0.0;
  for (int j = 0; j < ny; ++j) tot += __shfl_sync(0xffffffffu, racc, j);
  return gauss ? -tot * sp.inv_2sxi2 : tot;
}

// Warp-cooperative float64 Poisson window (one window per warp): lane i owns
// column factor I0 Ex_i / bg, lane j row j; row j is summed in column order
// by lane j and the rows in row order — bit-identical to
// loglik_poisson64_generic. All lanes return the value.
__device__ __forceinline__ double loglik_poisson64_warp(const PixView& pv, float x, float y,
                                                        float i0, const Spot& sp, int lane) {
  if (!(x == x) || !(y == y) || !(i0 == i0)) return nan_ll();
  int xlo, xhi, ylo, yhi;
  window_axis_f(x, sp.hw, pv.W, xlo, xhi);
  window_axis_f(y, sp.hw, pv.H, ylo, yhi);
  const int nx = xhi - xlo + 1, ny = yhi - ylo + 1;
  if (nx > 32 || ny > 32) return loglik_poisson64_generic(pv, x, y, i0, sp);
  const double a0 = (double)i0 / sp.bg64;
  const double colf = (lane < nx) ? a0 * psf_pixel64(xlo + lane, (double)x, sp) : 0.0;
  const double rowf = (lane < ny) ? psf_pixel64(ylo + lane, (double)y, sp) : 0.0;
  const float* row = pv.row(ylo + min(lane, ny - 1), xlo);
  double racc = 0.0;
  for (int i = 0; i < nx; ++i) {
    const double ci = __shfl_sync(0xffffffffu, colf, i);
    if (lane < ny) racc += poisson_term64((double)row[i], ci * rowf, sp.bg64);
  }
  double tot = 0.0;
  for (int j = 0; j < ny; ++j) tot += __shfl_sync(0xffffffffu, racc, j);
  return tot;
}

// One row of one window: the float64 partial row_j of the canonical form
// (column order), computed by one thread. Summing the rows of a window in row
// order reproduces loglik_gauss / loglik_poisson bit for bit.
__device__ __forceinline__ double loglik_row(const PixView& pv, float x, float y, float i0,
                                             const Spot& sp, int xlo, int nx, int yy) {
  const bool gauss = (sp.model == 0);
  const float inv_bg = 1.0f / sp.bg;
  const bool fast = !gauss && poisson_fast_ok(i0, sp);
  float d = pix_off(yy, y);
  float rowf = gauss ? expf(-(d * d) * sp.inv2s2) : psf_pixel(yy, y, sp);
  const float* row = pv.row(yy, xlo);
  double racc = 0.0;
  float racc_f = 0.0f;
  for (int i = 0; i < nx; ++i) {
    float dx = pix_off(xlo + i, x);
    if (gauss) {
      float ag = i0 * expf(-(dx * dx) * sp.inv2s2);
      float r = row[i] - fmaf(ag, rowf, sp.bg);
      racc = fma((double)r, (double)r, racc);
    } else {
      float ex = i0 * psf_pixel(xlo + i, x, sp) * inv_bg;
      racc_f += fast ? poisson_term<true>(row[i], ex * rowf, sp.bg)
                     : poisson_term<false>(row[i], ex * rowf, sp.bg);
    }
  }
  return gauss ? racc : (double)racc_f;
}

// window bounds of a state (for staging decisions)
__device__ __forceinline__ void window_of(float x, float y, const Spot& sp, i64 H, i64 W, int& xlo,
                                          int& xhi, int& ylo, int& yhi) {
  window_axis_f(x, sp.hw, W, xlo, xhi);
  window_axis_f(y, sp.hw, H, ylo, yhi);
}

template <int MAXS>
__global__ void __launch_bounds__(256) k_loglik(const float* __restrict__ pix, i64 H, i64 W,
                                                const float* __restrict__ xs,
                                                const float* __restrict__ ys,
                                                const float* __restrict__ is, i64 n, Spot sp,
                                                double* __restrict__ out) {
  const PixView pv = frame_view(pix, H, W);
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    out[i] = loglik_dispatch<MAXS>(pv, __ldg(xs + i), __ldg(ys + i), __ldg(is + i), sp);
}

// ---- float64 drop-in operator: spot_window_ssd (_speedups.pyx:42-83) ------
// Same operation order as the Cython loop, FMA contraction disabled.
__global__ void __launch_bounds__(128) k_ssd_f64(const double* __restrict__ pix, i64 H, i64 W,
                                                 const double* __restrict__ xs,
                                                 const double* __restrict__ ys,
                                                 const double* __restrict__ is, i64 n,
                                                 double inv2s2, double bg, int hw,
                                                 double* __restrict__ out) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    double x0 = xs[i], y0 = ys[i], amp = is[i];
    int xlo, xhi, ylo, yhi;
    window_axis(x0, hw, W, xlo, xhi);
    window_axis(y0, hw, H, ylo, yhi);
    double ssd = 0.0;
    for (int yy = ylo; yy <= yhi; ++yy) {
      double d = __dsub_rn((double)yy, y0);
      double gyv = exp(__dmul_rn(__dmul_rn(-d, d), inv2s2));
      const double* row = pix + (i64)yy * W;
      for (int xx = xlo; xx <= xhi; ++xx) {
        double dx = __dsub_rn((double)xx, x0);
        double gx = exp(__dmul_rn(__dmul_rn(-dx, dx), inv2s2));
        double pred = __dadd_rn(__dmul_rn(__dmul_rn(amp, gx), gyv), bg);
        double r = __dsub_rn(row[xx], pred);
        ssd = __dadd_rn(ssd, __dmul_rn(r, r));
      }
    }
    out[i] = ssd;
  }
}

}  // namespace pcs
