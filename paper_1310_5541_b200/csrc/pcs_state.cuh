// pcs_state.cuh — Philox replay, initial cloud, propagation (+ resampling
// gather), plain gather.
//
// Reference: state.py:115-127 (propagate_array), state.py:164-175
// (init_particle_set), filtering.py:107 (states[idx]).
#pragma once
#include "pcs_common.cuh"

namespace pcs {

struct Dyn {
  double sp, sv, si, dt;
};

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
//   x'  = RN32( RN( RN(x + RN(vx*dt)) + RN(z0*sp) ) )
//   vx' = RN32( RN(vx + RN(z2*sv)) )
//   I0' = max( RN32( RN(I0 + RN(z4*si)) ), 0 )
// evaluated in float64 on the float32 inputs with FMA contraction disabled,
// exactly the operation sequence numpy performs on the upcast values.
__device__ __forceinline__ void propagate_one(const float in[5], const float z[5], const Dyn& d,
                                              float out[5]) {
  double x = (double)in[0], y = (double)in[1], vx = (double)in[2], vy = (double)in[3],
         i0 = (double)in[4];
  double x1 = __dadd_rn(x, __dmul_rn(vx, d.dt));
  double y1 = __dadd_rn(y, __dmul_rn(vy, d.dt));
  out[0] = __double2float_rn(__dadd_rn(x1, __dmul_rn((double)z[0], d.sp)));
  out[1] = __double2float_rn(__dadd_rn(y1, __dmul_rn((double)z[1], d.sp)));
  out[2] = __double2float_rn(__dadd_rn(vx, __dmul_rn((double)z[2], d.sv)));
  out[3] = __double2float_rn(__dadd_rn(vy, __dmul_rn((double)z[3], d.sv)));
  float iv = __double2float_rn(__dadd_rn(i0, __dmul_rn((double)z[4], d.si)));
  out[4] = (iv > 0.0f) ? iv : ((iv == iv) ? 0.0f : iv);   // np.maximum(., 0) (NaN propagates)
}

template <bool GATHER>
__global__ void __launch_bounds__(256) k_propagate(const float* __restrict__ sin,
                                                   float* __restrict__ sout, i64 ld, i64 n,
                                                   const int* __restrict__ anc, Dyn dyn, u64 seed,
                                                   u32 frame, i64 off) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    i64 src = GATHER ? (i64)__ldg(anc + i) : i;
    float s[5], z[5], o[5];
#pragma unroll
    for (int c = 0; c < 5; ++c) s[c] = __ldg(sin + c * ld + src);
    philox_normals5(seed, frame, (u64)(off + i), z);
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
