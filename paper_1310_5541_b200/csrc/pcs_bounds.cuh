// pcs_bounds.cuh — the appendix's mid-point approximation bound study on
// the device (bounds.py:116-180, experiments.py:370-388; SURVEY §8(f) rank
// 4): dense sampling of the second-derivative maxima (derivative_maxima) and
// the tensor Gauss-Legendre quadrature of the per-cell mid-point error
// (midpoint_error). Fields are the reference's built-ins in parametric form:
//   kind 0  a x^2 + b y^2 + c x + d y + e        (quadratic, linear, constant, x^2)
//   kind 1  sin(x) sin(y)                          (sinsin_field)
//   kind 2  i0 exp(-((x-x0)^2 + (y-y0)^2)/(2 s^2)) + i_bg   (gaussian_spot_field)
// in float64 with the reference's operation order per point.
#pragma once
#include "pcs_common.cuh"

namespace pcs {

struct FieldDev {
  int kind;
  double p[6];
};

__device__ __forceinline__ double gauss_core(const FieldDev& F, double x, double y) {
  // p = (i0, i_bg, x0, y0, s2)
  const double dx = __dsub_rn(x, F.p[2]), dy = __dsub_rn(y, F.p[3]);
  const double q = -__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
  return __dmul_rn(F.p[0], exp(__ddiv_rn(q, __dmul_rn(2.0, F.p[4]))));
}

__device__ __forceinline__ double field_f(const FieldDev& F, double x, double y) {
  if (F.kind == 0) {
    double v = __dadd_rn(__dmul_rn(F.p[0], __dmul_rn(x, x)), __dmul_rn(F.p[1], __dmul_rn(y, y)));
    v = __dadd_rn(v, __dmul_rn(F.p[2], x));
    v = __dadd_rn(v, __dmul_rn(F.p[3], y));
    return __dadd_rn(v, F.p[4]);
  }
  if (F.kind == 1) return __dmul_rn(sin(x), sin(y));
  return __dadd_rn(gauss_core(F, x, y), F.p[1]);
}

__device__ __forceinline__ void field_d2(const FieldDev& F, double x, double y, double& fxx,
                                         double& fyy) {
  if (F.kind == 0) {
    fxx = __dmul_rn(2.0, F.p[0]);
    fyy = __dmul_rn(2.0, F.p[1]);
  } else if (F.kind == 1) {
    fxx = __dmul_rn(-sin(x), sin(y));
    fyy = fxx;
  } else {
    const double c = gauss_core(F, x, y), s2 = F.p[4];
    const double dx = __dsub_rn(x, F.p[2]), dy = __dsub_rn(y, F.p[3]);
    fxx = __ddiv_rn(__dmul_rn(c, __dsub_rn(__ddiv_rn(__dmul_rn(dx, dx), s2), 1.0)), s2);
    fyy = __ddiv_rn(__dmul_rn(c, __dsub_rn(__ddiv_rn(__dmul_rn(dy, dy), s2), 1.0)), s2);
  }
}

// np.linspace(lo, hi, n)[i]: i * step + lo, the last point exactly hi
__device__ __forceinline__ double linspace_at(double lo, double hi, i64 n, i64 i) {
  if (n == 1) return lo;
  if (i == n - 1) return hi;
  const double step = __ddiv_rn(__dsub_rn(hi, lo), (double)(n - 1));
  return __dadd_rn(__dmul_rn((double)i, step), lo);
}

// max |f_xx|, max |f_yy| over the nx x ny sampling grid (bit patterns of
// non-negative doubles order like unsigned integers: exact, order-free)
__global__ void k_deriv_max(FieldDev F, double x_lo, double x_hi, i64 nx, double y_lo, double y_hi,
                            i64 ny, unsigned long long* out2) {
  unsigned long long mx = 0ull, my = 0ull;
  const i64 total = nx * ny;
  for (i64 k = blockIdx.x * (i64)blockDim.x + threadIdx.x; k < total;
       k += (i64)gridDim.x * blockDim.x) {
    const i64 iy = k / nx, ix = k - iy * nx;
    double fxx, fyy;
    field_d2(F, linspace_at(x_lo, x_hi, nx, ix), linspace_at(y_lo, y_hi, ny, iy), fxx, fyy);
    mx = max(mx, (unsigned long long)__double_as_longlong(fabs(fxx)));
    my = max(my, (unsigned long long)__double_as_longlong(fabs(fyy)));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    my = max(my, __shfl_xor_sync(0xffffffffu, my, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(out2, mx);
    atomicMax(out2 + 1, my);
  }
}

// signed mid-point error of every cell: integral over the cell of
// f - f(midpoint) by Q x Q tensor Gauss-Legendre quadrature (nodes / weights
// of np.polynomial.legendre.leggauss). One warp per cell; lane l sums the
// nodes a = l, l + 32, ... of every row b in a fixed order, then a fixed
// butterfly adds the lanes (deterministic).
__global__ void __launch_bounds__(256) k_midpoint_error(FieldDev F, const double* __restrict__ xe,
                                                        i64 ncols, const double* __restrict__ ye,
                                                        i64 nrows, const double* __restrict__ nodes,
                                                        const double* __restrict__ wts, int Q,
                                                        double* __restrict__ cell_err) {
  const int lane = threadIdx.x & 31;
  const i64 warps = (i64)gridDim.x * (blockDim.x / 32);
  for (i64 c = blockIdx.x * (i64)(blockDim.x / 32) + (threadIdx.x >> 5); c < ncols * nrows;
       c += warps) {
    const i64 j = c / ncols, i = c - j * ncols;
    const double x0 = xe[i], x1 = xe[i + 1], y0 = ye[j], y1 = ye[j + 1];
    const double w = __dsub_rn(x1, x0), h = __dsub_rn(y1, y0);
    const double hw = __ddiv_rn(w, 2.0), hh = __ddiv_rn(h, 2.0);
    const double fm = field_f(F, __ddiv_rn(__dadd_rn(x0, x1), 2.0), __ddiv_rn(__dadd_rn(y0, y1), 2.0));
    double acc = 0.0;
    for (int b = 0; b < Q; ++b) {
      const double py = __dadd_rn(y0, __dmul_rn(__dadd_rn(nodes[b], 1.0), hh));
      const double wy = __dmul_rn(wts[b], hh);
      double row = 0.0;
      for (int a = lane; a < Q; a += 32) {
        const double px = __dadd_rn(x0, __dmul_rn(__dadd_rn(nodes[a], 1.0), hw));
        const double wx = __dmul_rn(wts[a], hw);
        row = fma(__dsub_rn(field_f(F, px, py), fm), wx, row);
      }
      acc = fma(row, wy, acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) cell_err[c] = acc;
  }
}

}  // namespace pcs
