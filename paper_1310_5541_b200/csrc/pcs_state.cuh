// pcs_state.cuh — Philox replay, initial cloud, propagation (+ resampling
// gather), plain gather.
//
// Reference: state.py:115-127 (propagate_array), state.py:164-175
// (init_particle_set), filtering.py:107 (states[idx]).
#pragma once
#include "pcs_common.cuh"

namespace pcs {

// propagation parameters as float32 pairs hi + lo (hi = RN32(p), lo =
// RN32(p - hi)): the products z * p keep ~48 bits of p, so the float32
// propagation tracks the reference's float64 one to the final rounding even
// for parameters such as 0.1 that float32 cannot hold
struct Dyn {
  float sp, sv, si, dt;          // hi parts
  float sp_lo, sv_lo, si_lo, dt_lo;
};
__host__ __forceinline__ Dyn make_dyn(double sp, double sv, double si, double dt) {
  Dyn d;
  d.sp = (float)sp;
  d.sv = (float)sv;
  d.si = (float)si;
  d.dt = (float)dt;
  d.sp_lo = (float)(sp - (double)d.sp);
  d.sv_lo = (float)(sv - (double)d.sv);
  d.si_lo = (float)(si - (double)d.si);
  d.dt_lo = (float)(dt - (double)d.dt);
  return d;
}

// ---- replay: the exact normals pcs_propagate consumes ----------------------
__global__ void k_philox_normals(u64 seed, u32 frame, i64 off, i64 n, float* __restrict__ out,
                                 i64 ld) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    float z[5];
    philox_normals5(seed, frame, (u64)(off + i), z);
#pragma unroll
    for (int c = 0; c < 5; ++c) out[c * ld + i] = z[c];
  }
}

__global__ void k_philox_init_normals(u64 seed, i64 off, i64 n, float* __restrict__ out, i64 ld) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    float z[2];
    philox_normals2_init(seed, (u64)(off + i), z);
    out[i] = z[0];
    out[ld + i] = z[1];
  }
}

__global__ void k_philox_init_uniforms(u64 seed, i64 off, i64 n, double* __restrict__ out, i64 ld) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    double u[2];
    philox_uniform2_init(seed, (u64)(off + i), u);
    out[i] = u[0];
    out[ld + i] = u[1];
  }
}

__global__ void k_philox_multinomial(u64 seed, u32 frame, i64 n, double* __restrict__ out) {
  for (i64 j = blockIdx.x * (i64)blockDim.x + threadIdx.x; j < n; j += (i64)gridDim.x * blockDim.x)
    out[j] = philox_multinomial_u(seed, frame, (u64)j);
}

// ---- init_particle_set (state.py:164-175) ----------------------------------
// point:   states = center
// uniform: x += RN(-half + RN(width * U))          (Generator.uniform = low + (high-low)*U)
// gauss:   x += RN(sigma * z)                      (Generator.normal  = loc + scale*z)
struct InitSpecDev {
  double c[5];
  int mode;
  double width, sigma;
};

__global__ void k_init(InitSpecDev spec, u64 seed, i64 off, i64 n, float* __restrict__ s, i64 ld) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    double x = spec.c[0], y = spec.c[1];
    if (spec.mode == 1) {
      double u[2];
      philox_uniform2_init(seed, (u64)(off + i), u);
      double half = spec.width / 2.0;
      x = __dadd_rn(x, __dadd_rn(-half, __dmul_rn(spec.width, u[0])));
      y = __dadd_rn(y, __dadd_rn(-half, __dmul_rn(spec.width, u[1])));
    } else if (spec.mode == 2) {
      float z[2];
      philox_normals2_init(seed, (u64)(off + i), z);
      x = __dadd_rn(x, __dmul_rn(spec.sigma, (double)z[0]));
      y = __dadd_rn(y, __dmul_rn(spec.sigma, (double)z[1]));
    }
    s[i] = __double2float_rn(x);
    s[ld + i] = __double2float_rn(y);
    s[2 * ld + i] = __double2float_rn(spec.c[2]);
    s[3 * ld + i] = __double2float_rn(spec.c[3]);
    s[4 * ld + i] = __double2float_rn(spec.c[4]);
  }
}

// ---- propagate (state.py:115-127), CANONICAL arithmetic --------------------
// float32 fused multiply-adds, each parameter p split as hi + lo (Dyn):
//   mul_add(a, p, b) = fma(a, p.hi, fma(a, p.lo, b))
//   x'  = mul_add(z0, sp, mul_add(vx, dt, x))     (old velocity, state.py:123-125)
//   vx' = mul_add(z2, sv, vx)
//   I0' = max(mul_add(z4, si, I0), 0)             (state.py:126; NaN propagates)
// The reference evaluates the same sums in float64 on float64 states; on
// the same float32 inputs the two agree to ~1 float32 ulp of the result
// (tests/test_gpu_stages.py). oracle.c orc_propagate restates this form
// bit-for-bit.
__device__ __forceinline__ float mul_add_split(float a, float hi, float lo, float b) {
  return __fmaf_rn(a, hi, __fmaf_rn(a, lo, b));
}
__device__ __forceinline__ void propagate_one(const float in[5], const float z[5], const Dyn& d,
                                              float out[5]) {
  out[0] = mul_add_split(z[0], d.sp, d.sp_lo, mul_add_split(in[2], d.dt, d.dt_lo, in[0]));
  out[1] = mul_add_split(z[1], d.sp, d.sp_lo, mul_add_split(in[3], d.dt, d.dt_lo, in[1]));
  out[2] = mul_add_split(z[2], d.sv, d.sv_lo, in[2]);
  out[3] = mul_add_split(z[3], d.sv, d.sv_lo, in[3]);
  const float iv = mul_add_split(z[4], d.si, d.si_lo, in[4]);
  out[4] = (iv > 0.0f) ? iv : ((iv == iv) ? 0.0f : iv);   // np.maximum(., 0) (NaN propagates)
}

template <bool GATHER>
__global__ void __launch_bounds__(256) k_propagate(const float* __restrict__ sin,
                                                   float* __restrict__ sout, i64 ld, i64 n,
                                                   const int* __restrict__ anc, Dyn dyn,
                                                   PhiloxKey pk, u32 frame, i64 off) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    i64 src = GATHER ? (i64)__ldg(anc + i) : i;
    float s[5], z[5], o[5];
#pragma unroll
    for (int c = 0; c < 5; ++c) s[c] = __ldg(sin + c * ld + src);
    philox_normals5k(pk, frame, (u64)(off + i), z);
    propagate_one(s, z, dyn, o);
#pragma unroll
    for (int c = 0; c < 5; ++c) sout[c * ld + i] = o[c];
  }
}

// replay form: normals supplied by the caller (z[c*ld + i]); used to run the
// device arithmetic on a reference's recorded draws (parity tests)
__global__ void __launch_bounds__(256) k_propagate_given(const float* __restrict__ sin,
                                                         float* __restrict__ sout, i64 ld, i64 n,
                                                         const int* __restrict__ anc, Dyn dyn,
                                                         const float* __restrict__ zin, i64 ldz) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    i64 src = anc ? (i64)__ldg(anc + i) : i;
    float s[5], z[5], o[5];
#pragma unroll
    for (int c = 0; c < 5; ++c) {
      s[c] = __ldg(sin + c * ld + src);
      z[c] = __ldg(zin + c * ldz + i);
    }
    propagate_one(s, z, dyn, o);
#pragma unroll
    for (int c = 0; c < 5; ++c) sout[c * ld + i] = o[c];
  }
}

__global__ void k_gather(const float* __restrict__ sin, float* __restrict__ sout, i64 ld, i64 n,
                         const int* __restrict__ anc) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    i64 src = __ldg(anc + i);
#pragma unroll
    for (int c = 0; c < 5; ++c) sout[c * ld + i] = __ldg(sin + c * ld + src);
  }
}

}  // namespace pcs
