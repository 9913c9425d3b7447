/*
 * oracle.c — TEST INFRASTRUCTURE ONLY (CPU checker; never shipped, never the
 * thing measured). Plain-C restatement of the arithmetic of the reference hot
 * path (/root/reference/pkg/src/pcsir, cited per function) plus the canonical
 * exact-sum conventions documented in DESIGN.md §3. Written independently of
 * the CUDA sources so that it can check them. Only tests/, smoke() and the
 * bench's cpu_baseline / --impl reference legs load it.
 *
 * Build: make -C oracle   (gcc -O2 -fPIC -shared -ffp-contract=off)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;
typedef __int128 i128;

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

#define FX_STATE 40
#define FX_WQ 62
#define FX_W2 120
#define FX_S 95
#define FX_CDF 120

/* ------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon et al., SC'11): counter c0..c3, key (k0,k1).  */
/* ------------------------------------------------------------------ */
static void philox(uint32_t c[4], uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0;
    uint32_t n1 = (uint32_t)p1;
    uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
    uint32_t n3 = (uint32_t)p0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

void orc_philox4x32(uint64_t seed, const uint32_t* ctr, int64_t n, uint32_t* out) {
  for (int64_t i = 0; i < n; ++i) {
    uint32_t c[4] = {ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3]};
    philox(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    memcpy(out + 4 * i, c, 16);
  }
}

static double u01_double(uint32_t a, uint32_t b) {
  return ((double)(a >> 5) * 67108864.0 + (double)(b >> 6)) * (1.0 / 9007199254740992.0);
}

/* float64 Box–Muller on the same 24-bit uniforms the device uses:
 * r = sqrt(-2 ln u1), angle 2 pi (u2 - 1/2) */
static void bm64(uint32_t a, uint32_t b, double* z0, double* z1) {
  double u1 = ((double)(a >> 8) + 0.5) * 5.9604644775390625e-8;
  double u2 = (double)(b >> 8) * 5.9604644775390625e-8;
  double r = sqrt(-2.0 * log(u1));
  double th = 2.0 * M_PI * (u2 - 0.5);
  *z0 = r * cos(th);
  *z1 = r * sin(th);
}

/* float64 Box–Muller on 22-bit u1 / 20-bit u2 (the propagation normals) */
static double bm_r22(uint32_t a) { return sqrt(-2.0 * log(((double)a + 0.5) * 2.384185791015625e-07)); }
static double bm_t20(uint32_t b) { return 2.0 * M_PI * ((double)b * 9.5367431640625e-07 - 0.5); }

/* the N x 5 standard normals of one propagation (state.py:125), out[c*n+i]:
 * one Philox block (x, y, z, w) per particle, three Box–Muller pairs
 * (pcs_common.cuh philox_normals5) */
void orc_propagate_normals(uint64_t seed, uint32_t frame, int64_t off, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    uint64_t idx = (uint64_t)(off + i);
    uint32_t c[4] = {(uint32_t)idx, (uint32_t)(idx >> 32), frame, (1u << 4) | 0u};
    philox(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    double r0 = bm_r22(c[0] >> 10), t0 = bm_t20(c[1] >> 12);
    double r1 = bm_r22(c[2] >> 10), t1 = bm_t20(c[3] >> 12);
    double r2 = bm_r22(((c[0] & 0x3FFu) << 12) | (c[1] & 0xFFFu));
    double t2 = bm_t20(((c[2] & 0x3FFu) << 10) | ((c[3] >> 2) & 0x3FFu));
    out[0 * n + i] = r0 * cos(t0);
    out[1 * n + i] = r0 * sin(t0);
    out[2 * n + i] = r1 * cos(t1);
    out[3 * n + i] = r1 * sin(t1);
    out[4 * n + i] = r2 * cos(t2);
  }
}

/* the two init normals (state.py:173), out[c*n+i] */
void orc_init_normals(uint64_t seed, int64_t off, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    uint64_t idx = (uint64_t)(off + i);
    uint32_t c[4] = {(uint32_t)idx, (uint32_t)(idx >> 32), 0u, (2u << 4)};
    philox(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    bm64(c[0], c[1], &out[i], &out[n + i]);
  }
}

/* systematic offset (filtering.py:99 rng.random()) */
double orc_resample_u(uint64_t seed, uint32_t frame) {
  uint32_t c[4] = {0u, 0u, frame, (3u << 4)};
  philox(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  return u01_double(c[0], c[1]);
}

/* multinomial points (filtering.py:97 rng.random(n)) */
void orc_multinomial_points(uint64_t seed, uint32_t frame, int64_t n, double* out) {
  for (int64_t j = 0; j < n; ++j) {
    uint32_t c[4] = {(uint32_t)j, (uint32_t)((uint64_t)j >> 32), frame, (4u << 4)};
    philox(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    out[j] = u01_double(c[0], c[1]);
  }
}

/* ------------------------------------------------------------------ */
/* exact fixed point                                                  */
/* ------------------------------------------------------------------ */
static u128 shround(uint64_t m, int s) { /* round(m * 2^s), ties to even */
  if (m == 0) return 0;
  if (s >= 0) return ((u128)m) << s;
  int r = -s;
  if (r > 64) return 0;
  if (r == 64) return (m > (1ull << 63)) ? 1 : 0;
  uint64_t q = m >> r, rem = m & ((1ull << r) - 1ull), half = 1ull << (r - 1);
  if (rem > half || (rem == half && (q & 1ull))) q += 1;
  return q;
}

static i128 fx32(float v, int F) {
  uint32_t b;
  memcpy(&b, &v, 4);
  uint32_t ef = (b >> 23) & 0xFF;
  uint64_t m = b & 0x7FFFFF;
  int e;
  if (ef == 0) {
    e = -149;
  } else {
    m |= 0x800000;
    e = (int)ef - 150;
  }
  i128 q = (i128)shround(m, e + F);
  return (b >> 31) ? -q : q;
}

static i128 fx64(double v, int F) {
  uint64_t b;
  memcpy(&b, &v, 8);
  uint32_t ef = (uint32_t)((b >> 52) & 0x7FF);
  uint64_t m = b & 0xFFFFFFFFFFFFFull;
  int e;
  if (ef == 0) {
    e = -1074;
  } else {
    m |= (1ull << 52);
    e = (int)ef - 1075;
  }
  i128 q = (i128)shround(m, e + F);
  return (b >> 63) ? -q : q;
}

/* correctly rounded (nearest-even) u128 -> double */
static double u128_to_double(u128 v) {
  if (v == 0) return 0.0;
  int nb = 128;
  while (!((v >> (nb - 1)) & 1)) --nb;
  if (nb <= 53) return (double)(uint64_t)v;
  int drop = nb - 53;
  u128 keep = v >> drop;
  u128 rem = v & ((((u128)1) << drop) - 1);
  u128 half = ((u128)1) << (drop - 1);
  if (rem > half || (rem == half && (keep & 1))) keep += 1;
  return ldexp((double)(uint64_t)keep, drop);
}

static double i128_to_double(i128 v) {
  return v < 0 ? -u128_to_double((u128)(-v)) : u128_to_double((u128)v);
}

/* value of round(v * 2^F) for inspection: out[0]=lo, out[1]=hi */
void orc_fixed_f32(const float* v, int64_t n, int F, uint64_t* out) {
  for (int64_t i = 0; i < n; ++i) {
    i128 q = fx32(v[i], F);
    out[2 * i] = (uint64_t)q;
    out[2 * i + 1] = (uint64_t)((u128)q >> 64);
  }
}

double orc_u128_to_double(uint64_t lo, uint64_t hi) {
  return u128_to_double(((u128)hi << 64) | lo);
}

/* ------------------------------------------------------------------ */
/* propagate_array (state.py:115-127) on float32 states with given     */
/* float32 normals, in the device's CANONICAL float32 form (pcs_state.cuh */
/* propagate_one): each parameter p split as hi = RN32(p), lo =          */
/* RN32(p - hi); mul_add(a, p, b) = fma(a, hi, fma(a, lo, b));           */
/*   x' = mul_add(z0, sp, mul_add(vx, dt, x)); vx' = mul_add(z2, sv, vx);*/
/*   I0' = max(mul_add(z4, si, I0), 0)                                  */
/* s, z, out: SoA [5][n]. (The reference's float64 sums, state.py:123-126,*/
/* agree to ~1 float32 ulp; orc_propagate_f64 below is numpy's order.)  */
/* ------------------------------------------------------------------ */
typedef struct { float hi, lo; } split32;
static split32 split_param(double p) {
  split32 s;
  s.hi = (float)p;
  s.lo = (float)(p - (double)s.hi);
  return s;
}
static float mul_add(float a, split32 p, float b) { return fmaf(a, p.hi, fmaf(a, p.lo, b)); }

void orc_propagate(const float* s, const float* z, int64_t n, double sp, double sv, double si,
                   double dt, float* out) {
  const split32 P = split_param(sp), V = split_param(sv), I = split_param(si), T = split_param(dt);
  for (int64_t i = 0; i < n; ++i) {
    float x = s[i], y = s[n + i], vx = s[2 * n + i], vy = s[3 * n + i], i0 = s[4 * n + i];
    out[i] = mul_add(z[i], P, mul_add(vx, T, x));
    out[n + i] = mul_add(z[n + i], P, mul_add(vy, T, y));
    out[2 * n + i] = mul_add(z[2 * n + i], V, vx);
    out[3 * n + i] = mul_add(z[3 * n + i], V, vy);
    float iv = mul_add(z[4 * n + i], I, i0);
    out[4 * n + i] = (iv > 0.0f) ? iv : ((iv == iv) ? 0.0f : iv);
  }
}

/* numpy's float64 order on the upcast float32 values, rounded once to   */
/* float32 (what the reference's propagate_array gives on these inputs) */
void orc_propagate_f64(const float* s, const float* z, int64_t n, double sp, double sv, double si,
                       double dt, float* out) {
  for (int64_t i = 0; i < n; ++i) {
    double x = s[i], y = s[n + i], vx = s[2 * n + i], vy = s[3 * n + i], i0 = s[4 * n + i];
    double x1 = x + vx * dt;
    double y1 = y + vy * dt;
    out[i] = (float)(x1 + (double)z[i] * sp);
    out[n + i] = (float)(y1 + (double)z[n + i] * sp);
    out[2 * n + i] = (float)(vx + (double)z[2 * n + i] * sv);
    out[3 * n + i] = (float)(vy + (double)z[3 * n + i] * sv);
    float iv = (float)(i0 + (double)z[4 * n + i] * si);
    out[4 * n + i] = (iv > 0.0f) ? iv : ((iv == iv) ? 0.0f : iv);
  }
}

/* ------------------------------------------------------------------ */
/* spot_window_ssd (_speedups.pyx:42-83), float64, same loop order      */
/* ------------------------------------------------------------------ */
void orc_spot_window_ssd(const double* pix, int64_t H, int64_t W, const double* xs,
                         const double* ys, const double* is, int64_t n, double sigma,
                         double bg, int64_t hw, double* out) {
  double inv = 1.0 / (2.0 * sigma * sigma);
  double* gx = (double*)malloc(sizeof(double) * (2 * hw + 1));
  double* gy = (double*)malloc(sizeof(double) * (2 * hw + 1));
  for (int64_t i = 0; i < n; ++i) {
    double x0 = xs[i], y0 = ys[i], amp = is[i];
    int64_t cx = (int64_t)floor(x0 + 0.5), cy = (int64_t)floor(y0 + 0.5);
    int64_t xlo = cx - hw, xhi = cx + hw, ylo = cy - hw, yhi = cy + hw;
    if (xlo < 0) xlo = 0; else if (xlo > W - 1) xlo = W - 1;
    if (xhi < 0) xhi = 0; else if (xhi > W - 1) xhi = W - 1;
    if (ylo < 0) ylo = 0; else if (ylo > H - 1) ylo = H - 1;
    if (yhi < 0) yhi = 0; else if (yhi > H - 1) yhi = H - 1;
    for (int64_t xi = xlo; xi <= xhi; ++xi) {
      double d = (double)xi - x0;
      gx[xi - xlo] = exp(-d * d * inv);
    }
    for (int64_t yi = ylo; yi <= yhi; ++yi) {
      double d = (double)yi - y0;
      gy[yi - ylo] = exp(-d * d * inv);
    }
    double ssd = 0.0;
    for (int64_t yi = ylo; yi <= yhi; ++yi) {
      double gyv = gy[yi - ylo];
      for (int64_t xi = xlo; xi <= xhi; ++xi) {
        double r = pix[yi * W + xi] - (amp * gx[xi - xlo] * gyv + bg);
        ssd += r * r;
      }
    }
    out[i] = ssd;
  }
  free(gx);
  free(gy);
}

/* Config-3 Poisson log-likelihood ratio (R19, new), float64:
 * model 1 erf pixel integral, model 2 mid-point 4x4. Brute force over the
 * 4x4 sub-pixels for model 1 (each sub-pixel integrated exactly), which
 * telescopes to the pixel integral the device evaluates. */
static double gauss_int(double a, double b, double sigma) { /* int_a^b exp(-t^2/2s^2) dt */
  double s2 = sqrt(2.0) * sigma;
  return sigma * sqrt(M_PI / 2.0) * (erf(b / s2) - erf(a / s2));
}

void orc_poisson_loglik(const double* pix, int64_t H, int64_t W, const double* xs,
                        const double* ys, const double* is, int64_t n, double sigma, double bg,
                        int64_t hw, int model, double* out) {
  double inv = 1.0 / (2.0 * sigma * sigma);
  for (int64_t i = 0; i < n; ++i) {
    double x0 = xs[i], y0 = ys[i], amp = is[i];
    int64_t cx = (int64_t)floor(x0 + 0.5), cy = (int64_t)floor(y0 + 0.5);
    int64_t xlo = cx - hw, xhi = cx + hw, ylo = cy - hw, yhi = cy + hw;
    if (xlo < 0) xlo = 0; else if (xlo > W - 1) xlo = W - 1;
    if (xhi < 0) xhi = 0; else if (xhi > W - 1) xhi = W - 1;
    if (ylo < 0) ylo = 0; else if (ylo > H - 1) ylo = H - 1;
    if (yhi < 0) yhi = 0; else if (yhi > H - 1) yhi = H - 1;
    double ll = 0.0;
    for (int64_t yi = ylo; yi <= yhi; ++yi) {
      for (int64_t xi = xlo; xi <= xhi; ++xi) {
        double mu = 0.0;
        for (int sy = 0; sy < 4; ++sy) {
          for (int sx = 0; sx < 4; ++sx) {
            if (model == 1) {
              double ax = (double)xi - 0.5 + 0.25 * sx - x0, ay = (double)yi - 0.5 + 0.25 * sy - y0;
              mu += gauss_int(ax, ax + 0.25, sigma) * gauss_int(ay, ay + 0.25, sigma);
            } else {
              double dx = (double)xi - 0.375 + 0.25 * sx - x0, dy = (double)yi - 0.375 + 0.25 * sy - y0;
              mu += exp(-dx * dx * inv) * exp(-dy * dy * inv) / 16.0;
            }
          }
        }
        mu *= amp;
        ll += pix[yi * W + xi] * log1p(mu / bg) - mu;
      }
    }
    out[i] = ll;
  }
}

/* ------------------------------------------------------------------ */
/* Canonical exact cdf and resampling (filtering.py:93-100 with an exact */
/* prefix in place of the sequential float64 cumsum)       */
/* ------------------------------------------------------------------ */
void orc_cdf_exact(const float* w, int64_t n, double* cdf) {
  u128 acc = 0;
  for (int64_t i = 0; i < n; ++i) {
    acc += (u128)fx32(w[i], FX_CDF);
    cdf[i] = ldexp(u128_to_double(acc), -FX_CDF);
  }
  if (n > 0) cdf[n - 1] = 1.0; /* filtering.py:95 */
}

/* searchsorted(cdf, (u + arange(n)) / n, side='right'); index n clamped */
void orc_systematic_from_cdf(const double* cdf, int64_t n, double u, int32_t* anc) {
  int64_t i = 0;
  for (int64_t j = 0; j < n; ++j) {
    double p = (u + (double)j) / (double)n;
    while (i < n && cdf[i] <= p) ++i;
    anc[j] = (int32_t)(i < n ? i : n - 1);
  }
}

void orc_searchsorted_right(const double* cdf, int64_t n, const double* pts, int64_t m,
                            int32_t* anc) {
  for (int64_t j = 0; j < m; ++j) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (cdf[mid] <= pts[j]) lo = mid + 1;
      else hi = mid;
    }
    anc[j] = (int32_t)(lo < n ? lo : n - 1);
  }
}

/* ------------------------------------------------------------------ */
/* Canonical per-bin dummies (binning.py:157-172): exact integer sums of */
/* round(s * 2^40) per bin; mean = RN32(RN64(RN64(S)/count) * 2^-40).   */
/* Weighted CoM: SW = sum round(w 2^62) round(s 2^40), SWq = sum round(w */
/* 2^62); mean = RN32(RN64(RN64(SW)/RN64(SWq)) * 2^-40).                 */
/* s: SoA [5][n] float32; out d: SoA [5][m].                             */
/* ------------------------------------------------------------------ */
void orc_dummies_exact(const float* s, int64_t n, const int32_t* bin_of, int64_t m,
                       const int64_t* counts, const float* prior_w, float* d) {
  i128* acc = (i128*)calloc((size_t)m * 6, sizeof(i128));
  for (int64_t i = 0; i < n; ++i) {
    int64_t b = bin_of[i];
    i128 wq = prior_w ? fx32(prior_w[i], FX_WQ) : 1;
    for (int c = 0; c < 5; ++c) acc[b * 6 + c] += fx32(s[c * n + i], FX_STATE) * wq;
    acc[b * 6 + 5] += wq;
  }
  for (int64_t b = 0; b < m; ++b) {
    double den = prior_w ? i128_to_double(acc[b * 6 + 5]) : (double)counts[b];
    for (int c = 0; c < 5; ++c) {
      double num = i128_to_double(acc[b * 6 + c]);
      d[c * m + b] = (float)ldexp(num / den, -FX_STATE);
    }
  }
  free(acc);
}

/* ------------------------------------------------------------------ */
/* Canonical normaliser (filtering.py:75-85 in the log domain):           */
/* m = max logw; S = sum round(exp(logw - m) 2^95); w = RN32(exp(.)/S64) */
/* returns 1 when degenerate (all -inf)                                  */
/* ------------------------------------------------------------------ */
int orc_normalize(const double* logw, int64_t n, float* w, double* m_out, double* s_out) {
  double m = -INFINITY;
  for (int64_t i = 0; i < n; ++i)
    if (logw[i] > m) m = logw[i];
  if (!(m > -INFINITY)) return 1;
  i128 S = 0;
  for (int64_t i = 0; i < n; ++i) S += fx64(exp(logw[i] - m), FX_S);
  double Sf = ldexp(i128_to_double(S), -FX_S);
  for (int64_t i = 0; i < n; ++i) w[i] = (float)(exp(logw[i] - m) / Sf);
  if (m_out) *m_out = m;
  if (s_out) *s_out = Sf;
  return 0;
}

/* Canonical estimate and ESS (filtering.py:88-90,112-114):
 * est_c = RN64(sum round(w 2^62) round(s 2^40)) 2^-102;
 * ESS = 1 / (RN64(sum round(w^2 2^120)) 2^-120). s SoA [5][n]. */
void orc_estimate_ess(const float* s, const float* w, int64_t n, double* est, double* ess) {
  i128 acc[5] = {0, 0, 0, 0, 0};
  i128 w2 = 0;
  for (int64_t i = 0; i < n; ++i) {
    i128 wq = fx32(w[i], FX_WQ);
    for (int c = 0; c < 5; ++c) acc[c] += wq * fx32(s[c * n + i], FX_STATE);
    w2 += fx64((double)w[i] * (double)w[i], FX_W2);
  }
  for (int c = 0; c < 5; ++c) est[c] = ldexp(i128_to_double(acc[c]), -(FX_WQ + FX_STATE));
  *ess = 1.0 / ldexp(i128_to_double(w2), -FX_W2);
}
