// pcs_track.cuh — fused SIR frame kernels (device-resident loop).
//
// One frame of sir_track (filtering.py:176-182, sis_step :62-72) with
// ResampleConfig(threshold_fraction=1.0, "systematic"): gather + propagate +
// per-particle likelihood -> max -> exact normaliser -> exact estimate/ESS ->
// decision -> exact-prefix systematic resampling (k_sys_resample).
// Canonical arithmetic is shared with pcSIR (pcs_fused.cuh) and with the
// general path, so pcSIR with one particle per cell equals SIR bit-for-bit.
#pragma once
#include "pcs_common.cuh"
#include "pcs_fused.cuh"
#include "pcs_lik.cuh"
#include "pcs_state.cuh"
#include "pcs_weights.cuh"

namespace pcs {

// frame region staged in shared memory by every CTA of the SIR likelihood
// kernel: SIR_SW x SIR_SW pixels centred on the previous estimate; particles
// whose window lies inside read it from shared memory, the others from HBM
// (same pixel values, identical log-likelihoods)
constexpr int SIR_SW = 64;

// log of a prior weight, out of line (only frames after a non-resampling frame)
__device__ __noinline__ double log_prior(float w) { return log((double)w); }

#ifndef PCS_SIR_MINB
#define PCS_SIR_MINB 2   // 2 CTAs / SM at 128 registers (1: 200-255 registers, 20-40 % slower)
#endif
template <int MAXS>
__global__ void __launch_bounds__(256, PCS_SIR_MINB) k_sir_propagate_lik(TrackParams P) {
  __shared__ __align__(128) float stg[SIR_SW * SIR_SW];
  __shared__ __align__(8) unsigned long long tma_bar;
  TrackCtl* C = P.ctl;
  const i64 k = C->k;
  const float* sin = (k & 1) ? P.buf1 : P.buf0;
  float* sout = (k & 1) ? P.buf0 : P.buf1;
  const float* frame = C->frames + (k - C->k_frames) * P.H * P.W;
  const PixView pv = frame_view(frame, P.H, P.W);
  PixView ps = pv;
  int sx0, sy0, sw, sh;
  if (C->fmap_ok) {
    // 64 x 64 region by TMA (4 boxes of 64 x 16; x origin 16-byte aligned;
    // pixels beyond the frame arrive as zeros and are never read)
    sw = SIR_SW;
    sh = SIR_SW;
    sx0 = (int)min(max((i64)floor(C->center[0]) - SIR_SW / 2, (i64)0), max(P.W - SIR_SW, (i64)0)) & ~3;
    sy0 = (int)min(max((i64)floor(C->center[1]) - SIR_SW / 2, (i64)0), max(P.H - SIR_SW, (i64)0));
    if (threadIdx.x == 0)
      tma_stage_issue(stg, P.fmap, sx0, sy0, (int)(k - C->k_frames), SIR_SW / FMAP_BY, &tma_bar);
    __syncthreads();
    tma_stage_wait(&tma_bar);
    sw = (int)min((i64)SIR_SW, P.W - sx0);   // valid columns / rows for the inside test
    sh = (int)min((i64)SIR_SW, P.H - sy0);
    ps.pitch = SIR_SW;
  } else {
    sw = (int)min((i64)SIR_SW, P.W);
    sh = (int)min((i64)SIR_SW, P.H);
    sx0 = (int)min(max((i64)floor(C->center[0]) - sw / 2, (i64)0), P.W - sw);
    sy0 = (int)min(max((i64)floor(C->center[1]) - sh / 2, (i64)0), P.H - sh);
    for (int p = threadIdx.x; p < sw * sh; p += blockDim.x)
      stg[p] = __ldg(frame + (i64)(sy0 + p / sw) * P.W + (sx0 + p % sw));
    __syncthreads();
    ps.pitch = sw;
  }
  ps.base = stg;
  ps.x0 = sx0;
  ps.y0 = sy0;
  long long lmax = LLONG_MIN;
  bool bad = false;
  const i64 n = P.n, ld = P.ld;
  const bool prior = C->prior_nonuniform != 0;
  // chunks of SIR_CHUNK particles: the first static, then dynamic tickets (a
  // CTA on a slower SM takes fewer chunks)
  // (P.sir_chunk == 0: plain grid stride, chunk = one block, no tickets)
  __shared__ long long s_next;
  const bool dyn = P.sir_chunk > 0;
  const i64 SIR_CHUNK = dyn ? P.sir_chunk : blockDim.x;
  const i64 nch = ceil_div(n, SIR_CHUNK);
  for (i64 ch = blockIdx.x; ch < nch;) {
    if (dyn && threadIdx.x == 0) s_next = gridDim.x + (long long)atomicAdd(&C->sir_ticket, 1u);
    for (i64 j = ch * SIR_CHUNK + threadIdx.x; j < min(n, (ch + 1) * SIR_CHUNK); j += blockDim.x) {
    i64 src = (i64)__ldg(P.anc + j);
    float s[5], z[5], o[5];
#pragma unroll
    for (int c = 0; c < 5; ++c) s[c] = __ldg(sin + c * ld + src);
    philox_normals5k(P.pk, P.frame0 + (u32)k, (u64)(P.idx_off + j), z);
    propagate_one(s, z, P.dyn, o);
#pragma unroll
    for (int c = 0; c < 5; ++c) sout[c * ld + j] = o[c];
    int xlo, xhi, ylo, yhi;
    window_axis_f(o[0], P.spot.hw, P.W, xlo, xhi);
    window_axis_f(o[1], P.spot.hw, P.H, ylo, yhi);
    const bool inside = xlo >= sx0 && xhi < sx0 + sw && ylo >= sy0 && yhi < sy0 + sh;
    PixView v = pv;
    v.base = inside ? ps.base : pv.base;
    v.pitch = inside ? ps.pitch : pv.pitch;
    v.x0 = inside ? ps.x0 : 0;
    v.y0 = inside ? ps.y0 : 0;
    double ll = loglik_dispatch<MAXS, false>(v, o[0], o[1], o[4], P.spot);
    // log w = log(w_prev) + ll (k_weight_update, binning.py:190-192 / filtering.py:69)
    if (prior) ll = __dadd_rn(log_prior(P.wprev[j]), ll);
    P.ll[j] = ll;
    if (!(ll == ll) || ll == INFINITY) bad = true;
    lmax = max(lmax, (long long)f64_to_ordered(ll));
    }
    if (dyn) {
      __syncthreads();
      ch = s_next;
      __syncthreads();   // s_next is rewritten at the top of the next chunk
    } else {
      ch += gridDim.x;
    }
  }
  if (dyn && threadIdx.x == 0 && atomicAdd(&C->sir_done, 1u) == gridDim.x - 1) {   // all drawn
    C->sir_ticket = 0;
    C->sir_done = 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lmax = max(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
  if ((threadIdx.x & 31) == 0) atomicMax((long long*)&C->max_ll_ord, lmax);
  if (bad) set_flag(C, PCS_FLAG_NONFINITE);
}

// pcSIR frame whose particles carry prior weights (threshold resampling, no
// resampling at the previous frame): per-particle log w = log(w_prev) +
// ll[cell] (binning.py:190-192, filtering.py:69) and its maximum; the SIR
// kernels below then normalise, estimate and resample per particle.
__global__ void __launch_bounds__(256) k_pc_prior_ll(TrackParams P) {
  TrackCtl* C = P.ctl;
  if (!C->pc_prior || (C->flags & PCS_FLAG_CAPACITY)) return;
  long long lmax = LLONG_MIN;
  bool bad = false;
  for (i64 j = blockIdx.x * (i64)blockDim.x + threadIdx.x; j < P.n; j += (i64)gridDim.x * blockDim.x) {
    const double ll = __dadd_rn(log_prior(P.wprev[j]), code_ll(P, P.pslot[j]));
    P.ll[j] = ll;
    if (!(ll == ll) || ll == INFINITY) bad = true;
    lmax = max(lmax, (long long)f64_to_ordered(ll));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lmax = max(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
  if ((threadIdx.x & 31) == 0) atomicMax((long long*)&C->max_ll_ord, lmax);
  if (bad) set_flag(C, PCS_FLAG_NONFINITE);
}

// S = sum round(exp(ll - m) * 2^95); leaves exp(ll - m) in P.ll
__global__ void __launch_bounds__(256) k_sir_sum(TrackParams P) {
  __shared__ i128 sh[8];
  TrackCtl* C = P.ctl;
  // pcSIR frame with uniform priors, or one the bins kernel could not hold
  if (P.method == 1 && (!C->pc_prior || (C->flags & PCS_FLAG_CAPACITY))) return;
  const double m = ordered_to_f64(C->max_ll_ord);
  i128 acc = 0;
  for (i64 j = blockIdx.x * (i64)blockDim.x + threadIdx.x; j < P.n; j += (i64)gridDim.x * blockDim.x) {
    const double ex = exp(__dsub_rn(P.ll[j], m));
    P.ll[j] = ex;   // from here on P.ll holds exp(ll - m) (one exp per particle per frame)
    acc += f64_to_fixed(ex, FX_S);
  }
  i128 t = block_sum_i128<256>(acc, sh);
  if (threadIdx.x == 0) atomic_add_i128(C->S, t);
}

// one thread: frame outputs, resampling decision, frame counter advance
__device__ __forceinline__ void sir_finalize(const TrackParams& P) {
  TrackCtl* C = P.ctl;
  const i64 k = C->k, ko = k - C->k_out;
  const bool row = k < C->k_end;   // (an output row exists for this frame)
  const double mf = ordered_to_f64(C->max_ll_ord);
  const bool degenerate = (mf == -INFINITY);
  const bool bad_m = !(mf == mf) || mf == INFINITY;
  double est[5];
  for (int c = 0; c < 5; ++c) {
    est[c] = scalbn(i128_to_f64_rn(load_i128(C->est[c])), -(FX_WQ + FX_STATE));
    if (row) C->out_est[ko * 5 + c] = est[c];
  }
  if (est[0] == est[0] && est[1] == est[1]) {   // staging window of the next frame
    C->center[0] = est[0];
    C->center[1] = est[1];
  }
  double ess = 1.0 / scalbn(i128_to_f64_rn(load_i128(C->w2)), -FX_W2);
  if (row) C->out_ess[ko] = ess;
  bool flag_bad = degenerate || bad_m;
  if (degenerate) set_flag(C, PCS_FLAG_DEGENERATE);
  if (bad_m) set_flag(C, PCS_FLAG_NONFINITE);
  int res = (!flag_bad && ess < P.thresh) ? 1 : 0;   // filtering.py:169-170
  // without resampling the next frame starts from these weights unless they
  // are all equal (then uniform, as the general driver does)
  C->prior_nonuniform = (!res && !flag_bad && C->wmin_bits != C->wmax_bits) ? 1 : 0;
  const i64 evals = (P.method == 1) ? C->frame_occ : P.n;   // pcSIR: one per occupied cell
  if (row) {
    C->out_res[ko] = (unsigned char)res;
    C->out_occ[ko] = evals;
  }
  C->evals += evals;
  C->do_resample = res;
  C->m = mf;
  C->Sf = scalbn(i128_to_f64_rn(load_i128(C->S)), -FX_S);
  C->u = philox_resample_u(P.seed, P.frame0 + (u32)k);
  C->res_frame = P.frame0 + (u32)k;
  reset_frame(C);
  C->k = k + 1;
}


// estimate / ESS numerators and the min/max normalised weight
__global__ void __launch_bounds__(256) k_sir_stats(TrackParams P) {
  __shared__ i128 sh[8];
  TrackCtl* C = P.ctl;
  if (P.method == 1 && (!C->pc_prior || (C->flags & PCS_FLAG_CAPACITY))) return;
  const i64 k = C->k;
  const float* st = (k & 1) ? P.buf0 : P.buf1;
  const double m = ordered_to_f64(C->max_ll_ord);
  const double Sf = scalbn(i128_to_f64_rn(load_i128(C->S)), -FX_S);
  const i64 n = P.n, ld = P.ld;
  i128 e[6] = {0, 0, 0, 0, 0, 0};
  bool range = false;
  unsigned wmin = 0xFFFFFFFFu, wmax = 0u;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    float w = weight_from_ex(P.ll[i], Sf);
    wmin = min(wmin, __float_as_uint(w));
    wmax = max(wmax, __float_as_uint(w));
    // w <= 1: round(w 2^62) <= 2^62 fits a signed 64-bit value; for
    // 2^-17 <= |v| < 2^23, round(v 2^40) = v 2^40 exactly and fits as well
    const long long wq = (long long)f32_to_fixed(w, FX_WQ);
#pragma unroll
    for (int c = 0; c < 5; ++c) {
      const float v = st[c * ld + i];
      if (fabsf(v) >= 16777216.0f) range = true;
      const float av = fabsf(v);
      if (av >= 7.62939453125e-06f && av < 8388608.0f)   // 2^-17 <= |v| < 2^23: exact, < 2^63
        e[c] += (i128)wq * (i128)__float2ll_rn(__fmul_rn(v, 1099511627776.0f));
      else
        e[c] += (i128)wq * f32_to_fixed(v, FX_STATE);
    }
    e[5] += f64_to_fixed((double)w * (double)w, FX_W2);
  }
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    i128 tt = block_sum_i128<256>(e[c], sh);
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
    __threadfence();   // this CTA's atomics are visible before it is counted
  }
  // the last CTA to finish runs the frame's finalisation (no extra launch)
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(&C->stats_done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    C->stats_done = 0;
    if (!P.sharded) sir_finalize(P);   // (sharded: after the all-reduce, pcs_shard.cuh)
  }
}

}  // namespace pcs
