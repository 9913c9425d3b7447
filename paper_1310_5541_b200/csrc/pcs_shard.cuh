// pcs_shard.cuh — particle-sharded giant filter (config 5).
//
// Rank r of P holds the global particles [r n, (r+1) n) and owns the output
// slots [r n, (r+1) n). Per frame, every step stream-ordered with fixed-size
// collectives and no host synchronisation (graph-capturable):
//   k_pc_step1 (local; Philox on global indices) -> local exact cell sums
//   k_shard_bbox       local occupied-cell box       -> box (all-reduce MAX)
//   k_shard_export     box-window cells -> 16 int64 limbs each, in a fixed
//                      wcap-cell buffer               -> limbs (all-reduce SUM)
//   k_shard_import + k_pc_cells + k_pc_bins   identical on every rank
//   k_sys_resample mode 1 + k_shard_total     exact rank weight total
//                                                     -> totals (all-gather)
//   k_shard_ranges     every rank's emitted slot range from the gathered
//                      totals (monotone systematic ancestors: contiguous)
//   k_sys_resample mode 2 (rank prefix)       ancestors of this rank's slots
//   k_shard_pack       own slots keep their ancestors in place; the head /
//                      tail slots owned by rank r-1 / r+1 are packed
//                      (states) into fixed bcap-slot buffers -> send/recv
//   k_shard_unpack     received states appended after the local particles
//                      (index n + q); their slots point at them
// ESS-threshold resampling (filtering.py:169-171): a frame whose particles
// carry prior weights finishes per particle (k_pc_prior_ll, k_sir_sum,
// k_sir_stats on the local particles) with three more fixed-size
// all-reduces — the max log-weight (MAX), the exact normaliser (SUM of
// limbs), the exact estimate / ESS numerators (SUM of limbs) with the weight
// range (MAX) — and every rank then runs the same finalisation
// (k_shard_prior_in). Frames without prior weights pass neutral values.
// Multinomial resampling (filtering.py:96-97,100): ancestors are not
// monotone, so slots fetch states from any rank. From the gathered totals
// every rank knows the global cdf's value at each rank boundary, hence the
// rank holding the ancestor of each of its slots (k_shard_route); requests
// (slot offsets, bcap per rank pair) and the answering states go through
// two fixed-size all-to-alls (k_shard_serve, k_shard_install). The owner
// regenerates the slot's Philox point and searches its part of the cdf.
// Only boundary states move (the weight-share imbalance between ranks, not
// the whole state); the limb all-reduce is exact and associative, so every
// result is identical for any P. Capacity checks (window > wcap, a range
// reaching past a neighbour, boundary > bcap) are evaluated identically on
// every rank from the same gathered totals, so all ranks raise together.
// The int128 per-cell sums travel as three 42-bit limbs so an int64
// all-reduce over up to 2^21 ranks cannot overflow.
#pragma once
#include "pcs_common.cuh"
#include "pcs_fused.cuh"
#include "pcs_track.cuh"

namespace pcs {

constexpr int LIMBS_PER_CELL = 16;   // count + 5 components x 3 limbs

// box = (-ix0, ix1, -iy0, iy1, local occupied cells): MAX-reducible
__global__ void k_shard_bbox(TrackParams P, i64* out) {
  __shared__ long long s[4];
  TrackCtl* C = P.ctl;
  const u32 m = C->n_occ;
  if (threadIdx.x == 0) {
    s[0] = LLONG_MIN;
    s[1] = LLONG_MIN;
    s[2] = LLONG_MIN;
    s[3] = LLONG_MIN;
  }
  __syncthreads();
  const u32 mm = min(m, (u32)MAXM);
  for (u32 b = threadIdx.x; b < mm; b += blockDim.x) {
    const u32 cell = P.hkey[P.occ[b]];   // (the occupied list holds table slots)
    long long ix = (long long)cell % P.grid.ncols, iy = (long long)cell / P.grid.ncols;
    atomicMax(&s[0], -ix);
    atomicMax(&s[1], ix);
    atomicMax(&s[2], -iy);
    atomicMax(&s[3], iy);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 0; q < 4; ++q) out[q] = s[q];
    out[4] = m;
    if (m > (u32)MAXM) set_flag(C, PCS_FLAG_CAPACITY);
  }
}

// the global window from the reduced box; false (and the capacity flag) if
// it does not fit the fixed limb buffer
__device__ __forceinline__ bool shard_window(const i64* box, i64 wcap, i64& x0, i64& y0, i64& nx,
                                             i64& ny) {
  x0 = -box[0];
  y0 = -box[2];
  nx = box[1] - x0 + 1;
  ny = box[3] - y0 + 1;
  return nx >= 1 && ny >= 1 && nx * ny <= wcap;
}

__global__ void k_shard_export(TrackParams P, const i64* __restrict__ box, i64 wcap,
                               i64* __restrict__ limbs) {
  i64 x0, y0, nx, ny;
  const bool ok = shard_window(box, wcap, x0, y0, nx, ny);
  if (blockIdx.x == 0 && threadIdx.x == 0 && !ok) set_flag(P.ctl, PCS_FLAG_CAPACITY);
  if (!ok) return;
  const i64 W = nx * ny;
  const u64 M42 = (1ull << 42) - 1ull;
  for (i64 q = blockIdx.x * (i64)blockDim.x + threadIdx.x; q < W; q += (i64)gridDim.x * blockDim.x) {
    i64 ix = x0 + q % nx, iy = y0 + q / nx;
    i64* L = limbs + q * LIMBS_PER_CELL;
    const u32 flat = (u32)(iy * P.grid.ncols + ix);
    const u32 slot = ht_find(P, flat);
    const u32 cnt = (slot != HT_EMPTY) ? P.tab_cnt[slot] : 0u;
    L[0] = cnt;
    for (int c = 0; c < 5; ++c) {
      i128 v = 0;
      if (cnt) {
        v = tab_load(P, c, slot);
        tab_zero(P, c, slot);
      }
      L[1 + 3 * c] = (i64)((u64)v & M42);
      L[2 + 3 * c] = (i64)((u64)(v >> 42) & M42);
      L[3 + 3 * c] = (i64)(v >> 84);   // arithmetic shift keeps the sign
    }
    if (cnt) P.tab_cnt[slot] = 0;
  }
}

// after the export: empty the occupied list (import rebuilds it from the
// global window). The local keys stay: a cell the rank holds keeps its table
// slot through the import (ht_insert finds the key before any free slot on
// its probe path), so the particles' step-1 cell codes stay valid; the bins
// kernel frees every slot of the global list at the end of the frame.
__global__ void k_shard_reset(TrackParams P) {
  if (threadIdx.x == 0 && blockIdx.x == 0) P.ctl->n_occ = 0;
}

__global__ void k_shard_import(TrackParams P, const i64* __restrict__ box, i64 wcap,
                               const i64* __restrict__ limbs) {
  i64 x0, y0, nx, ny;
  if (!shard_window(box, wcap, x0, y0, nx, ny)) return;
  const i64 W = nx * ny;
  TrackCtl* C = P.ctl;
  for (i64 q = blockIdx.x * (i64)blockDim.x + threadIdx.x; q < W; q += (i64)gridDim.x * blockDim.x) {
    const i64* L = limbs + q * LIMBS_PER_CELL;
    i64 cnt = L[0];
    if (!cnt) continue;
    i64 ix = x0 + q % nx, iy = y0 + q / nx;
    const u32 flat = (u32)(iy * P.grid.ncols + ix);
    const u32 slot = ht_insert(P, flat);
    if (slot == HT_EMPTY) {
      set_flag(C, PCS_FLAG_CAPACITY);
      continue;
    }
    P.tab_cnt[slot] = (u32)cnt;
    for (int c = 0; c < 5; ++c) {
      i128 v = (i128)L[1 + 3 * c] + ((i128)L[2 + 3 * c] << 42) + ((i128)L[3 + 3 * c] << 84);
      tab_store(P, c, slot, v);
    }
    u32 idx = atomicAdd(&C->n_occ, 1u);
    if (idx < (u32)MAXM) P.occ[idx] = slot;
  }
}

__device__ __forceinline__ void u128_to_limbs(u128 v, i64* out) {
  const u64 M42 = (1ull << 42) - 1ull;
  out[0] = (i64)((u64)v & M42);
  out[1] = (i64)((u64)(v >> 42) & M42);
  out[2] = (i64)(u64)(v >> 84);
}
__device__ __forceinline__ u128 limbs_to_u128(const i64* L) {
  return (u128)(u64)L[0] + ((u128)(u64)L[1] << 42) + ((u128)(u64)L[2] << 84);
}

__device__ __forceinline__ void i128_to_limbs(i128 v, i64* out) {
  const u64 M42 = (1ull << 42) - 1ull;
  out[0] = (i64)((u64)v & M42);
  out[1] = (i64)((u64)(v >> 42) & M42);
  out[2] = (i64)(v >> 84);   // arithmetic shift keeps the sign
}
__device__ __forceinline__ i128 limbs_to_i128(const i64* L) {
  return (i128)L[0] + ((i128)L[1] << 42) + ((i128)L[2] << 84);
}
__device__ __forceinline__ void store_i128(u64* p, i128 v) {
  p[0] = (u64)v;
  p[1] = (u64)((u128)v >> 64);
}

// exact rank weight total = sum of the per-CTA totals of k_sys_resample mode 1
// (per-cell weights: nagg1 CTAs; prior-weight frames, per particle: nagg2)
__global__ void k_shard_total(TrackParams P, int nagg1, int nagg2, i64* __restrict__ total) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int nagg = P.ctl->pc_prior ? nagg2 : nagg1;
  u128 t = 0;
  if (P.ctl->do_resample)
    for (int c = 0; c < nagg; ++c) t += P.cta_agg[c];
  u128_to_limbs(t, total);
}

// ---- frames with prior weights: the all-reduced per-particle stages ----
// stage 0: local max log-weight (k_pc_prior_ll)     -> out[0]           (MAX)
// stage 1: local exact normaliser (k_sir_sum)        -> out[0..3) limbs  (SUM)
// stage 2: local estimate / ESS numerators (k_sir_stats) -> out[0..18) limbs (SUM),
//          weight range -> mm = (-wmin bits, wmax bits)                  (MAX)
// Frames without prior weights write neutral values.
__global__ void k_shard_prior_out(TrackParams P, int stage, i64* __restrict__ out,
                                  i64* __restrict__ mm) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const TrackCtl* C = P.ctl;
  const bool on = C->pc_prior != 0;
  if (stage == 0) {
    out[0] = on ? C->max_ll_ord : LLONG_MIN;
  } else if (stage == 1) {
    u128_to_limbs(on ? (u128)load_i128(C->S) : (u128)0, out);
  } else {
    for (int c = 0; c < 5; ++c) i128_to_limbs(on ? load_i128(C->est[c]) : (i128)0, out + 3 * c);
    i128_to_limbs(on ? load_i128(C->w2) : (i128)0, out + 15);
    mm[0] = on ? -(i64)C->wmin_bits : -(i64)0xFFFFFFFFll;
    mm[1] = on ? (i64)C->wmax_bits : 0;
  }
}

// install the reduced values; stage 2 then finalises the frame on every rank
// (the same inputs everywhere: the same decision, offset and outputs)
__global__ void k_shard_prior_in(TrackParams P, int stage, const i64* __restrict__ in,
                                 const i64* __restrict__ mm) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  TrackCtl* C = P.ctl;
  if (!C->pc_prior || (C->flags & PCS_FLAG_CAPACITY)) return;   // (as k_sir_stats)
  if (stage == 0) {
    C->max_ll_ord = in[0];
  } else if (stage == 1) {
    store_i128(C->S, (i128)limbs_to_u128(in));
  } else {
    for (int c = 0; c < 5; ++c) store_i128(C->est[c], limbs_to_i128(in + 3 * c));
    store_i128(C->w2, limbs_to_i128(in + 15));
    C->wmin_bits = (u32)(-mm[0]);
    C->wmax_bits = (u32)mm[1];
    sir_finalize(P);
  }
}

// every rank's emitted slot range [lo_q, hi_q) from the gathered totals,
// this rank's prefix / range / boundary counts, and the capacity checks
// (the same on every rank: same inputs)
// multi (multinomial): only this rank's exact prefix and bnd[q] = the global
// cdf's value at the last particle of rank q - 1, q = 1..world-1
__global__ void k_shard_ranges(TrackParams P, const i64* __restrict__ totals, int rank, int world,
                               i64 bcap, int multi, double* __restrict__ bnd) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  TrackCtl* C = P.ctl;
  const i64 n = P.n, ng = P.n_global;
  if (multi) {
    u128 pre = 0;
    for (int q = 0; q < world; ++q) {
      if (q == rank) {
        C->rank_prefix[0] = (u64)pre;
        C->rank_prefix[1] = (u64)(pre >> 64);
      }
      if (q > 0) bnd[q] = cdf_round(pre);
      pre += limbs_to_u128(totals + 3 * q);
    }
    return;
  }
  if (!C->do_resample) {
    C->rank_prefix[0] = C->rank_prefix[1] = 0;
    C->shard_lo = (i64)rank * n;
    C->shard_hi = (i64)(rank + 1) * n;
    C->shard_send[0] = C->shard_send[1] = 0;
    C->shard_recv[0] = C->shard_recv[1] = 0;
    return;
  }
  const double u = C->u, nd = (double)ng, eps = nd * 8.881784197001252e-16;
  u128 pre = 0;
  i64 lo_q = 0;
  bool bad = false;
  i64 lo_r = 0, hi_r = 0, hi_prev = 0, lo_next = ng;
  for (int q = 0; q < world; ++q) {
    const u128 tq = limbs_to_u128(totals + 3 * q);
    const u128 pnext = pre + tq;
    const i64 hi_q = (q == world - 1) ? ng : first_slot_fast(cdf_round(pnext), u, ng, nd, eps);
    // ranges reach at most into the neighbouring ranks' slots; boundary
    // chunks fit the exchange buffers; the range fits the ancestor buffer
    const i64 own0 = (i64)q * n, own1 = (i64)(q + 1) * n;
    if (lo_q < own0 - n || hi_q > own1 + n || hi_q - lo_q > P.slot_cap) bad = true;
    if (max((i64)0, min(hi_q, own0) - lo_q) > bcap || max((i64)0, hi_q - max(lo_q, own1)) > bcap)
      bad = true;
    if (q == rank) {
      C->rank_prefix[0] = (u64)pre;
      C->rank_prefix[1] = (u64)(pre >> 64);
      lo_r = lo_q;
      hi_r = hi_q;
    }
    if (q == rank - 1) hi_prev = hi_q;
    if (q == rank + 1) lo_next = lo_q;
    pre = pnext;
    lo_q = hi_q;
  }
  const i64 own0 = (i64)rank * n, own1 = (i64)(rank + 1) * n;
  C->shard_lo = lo_r;
  C->shard_hi = hi_r;
  C->shard_send[0] = max((i64)0, min(hi_r, own0) - lo_r);
  C->shard_send[1] = max((i64)0, hi_r - max(lo_r, own1));
  C->shard_recv[0] = (rank > 0) ? max((i64)0, hi_prev - own0) : 0;
  C->shard_recv[1] = (rank < world - 1) ? max((i64)0, own1 - lo_next) : 0;
  if (bad) set_flag(C, PCS_FLAG_CAPACITY);
}

// boundary buffers: float32 [5][bcap] + one slot holding the count (int bits)
__device__ __forceinline__ void put_count(float* buf, i64 bcap, i64 cnt) {
  buf[5 * bcap] = __int_as_float((int)cnt);
}
__device__ __forceinline__ i64 get_count(const float* buf, i64 bcap) {
  return (i64)__float_as_int(buf[5 * bcap]);
}

// no resampling: identity ancestors; the particles keep their normalised
// weights when they are not all equal (filtering.py:171)
__device__ __forceinline__ void shard_identity(const TrackParams& P, const TrackCtl* C, i64 tid,
                                               i64 nthr) {
  const bool keep = C->prior_nonuniform && !(C->flags & PCS_FLAG_CAPACITY);
  const bool prior = C->pc_prior != 0;
  const double Sf = C->Sf;
  for (i64 i = tid; i < P.n; i += nthr) {
    P.anc[i] = (int)i;
    if (keep) P.wprev[i] = prior ? weight_from_ex(P.ll[i], Sf) : code_wtab(P, P.pslot[i]);
  }
}

// own slots keep their ancestors (the next frame's gather indices); head /
// tail slots of the neighbours are packed as states
__global__ void k_shard_pack(TrackParams P, int rank, float* __restrict__ send_prev,
                             float* __restrict__ send_next, i64 bcap) {
  TrackCtl* C = P.ctl;
  const i64 n = P.n, ld = P.ld;
  const float* cur = (C->k & 1) ? P.buf1 : P.buf0;   // this frame's propagated states
  const i64 tid = blockIdx.x * (i64)blockDim.x + threadIdx.x, nthr = (i64)gridDim.x * blockDim.x;
  const bool cap = (C->flags & PCS_FLAG_CAPACITY) != 0;
  if (!C->do_resample || cap) {   // identity ancestors, nothing to send
    shard_identity(P, C, tid, nthr);
    if (tid == 0) {
      put_count(send_prev, bcap, 0);
      put_count(send_next, bcap, 0);
    }
    return;
  }
  const i64 lo = C->shard_lo, hi = C->shard_hi;
  const i64 own0 = (i64)rank * n, own1 = own0 + n;
  for (i64 s = tid; s < hi - lo; s += nthr) {
    const i64 j = lo + s;
    const int src = P.anc_out[s];
    if (j < own0) {
#pragma unroll
      for (int c = 0; c < 5; ++c) send_prev[c * bcap + (j - lo)] = cur[c * ld + src];
    } else if (j >= own1) {
#pragma unroll
      for (int c = 0; c < 5; ++c) send_next[c * bcap + (j - own1)] = cur[c * ld + src];
    } else {
      P.anc[j - own0] = src;
    }
  }
  if (tid == 0) {
    put_count(send_prev, bcap, C->shard_send[0]);
    put_count(send_next, bcap, C->shard_send[1]);
  }
}

// the received boundary states go after the local particles (index n + q,
// n + bcap + q) of the next frame's input; the slots they fill point at them
__global__ void k_shard_unpack(TrackParams P, const float* __restrict__ recv_prev,
                               const float* __restrict__ recv_next, i64 bcap) {
  TrackCtl* C = P.ctl;
  if (!C->do_resample || (C->flags & PCS_FLAG_CAPACITY)) return;
  const i64 n = P.n, ld = P.ld;
  float* cur = (C->k & 1) ? P.buf1 : P.buf0;
  const i64 cp = C->shard_recv[0], cn = C->shard_recv[1];
  const i64 tid = blockIdx.x * (i64)blockDim.x + threadIdx.x, nthr = (i64)gridDim.x * blockDim.x;
  if (tid == 0 && ((cp && get_count(recv_prev, bcap) != cp) || (cn && get_count(recv_next, bcap) != cn)))
    set_flag(C, PCS_FLAG_CAPACITY);   // (a protocol mismatch; cannot happen with one plan)
  for (i64 q = tid; q < cp; q += nthr) {
#pragma unroll
    for (int c = 0; c < 5; ++c) cur[c * ld + n + q] = recv_prev[c * bcap + q];
    P.anc[q] = (int)(n + q);
  }
  for (i64 q = tid; q < cn; q += nthr) {
#pragma unroll
    for (int c = 0; c < 5; ++c) cur[c * ld + n + bcap + q] = recv_next[c * bcap + q];
    P.anc[n - cn + q] = (int)(n + bcap + q);
  }
}

// ---- multinomial exchange ----
// first index in [0, n) of the rank's part of the global cdf with cdf > p
// (searchsorted 'right'), clamped to n - 1
__device__ __forceinline__ i64 local_search(const double* __restrict__ cdf, i64 n, double p) {
  i64 lo = 0, hi = n;
  while (lo < hi) {
    const i64 mid = (lo + hi) >> 1;
    if (__ldg(cdf + mid) <= p) lo = mid + 1;
    else hi = mid;
  }
  return lo < n ? lo : n - 1;
}

// slot j (global rank * n + local) draws p_j = philox_multinomial_u(seed, frame,
// j); its ancestor lives on rank q = #{q' >= 1 : bnd[q'] <= p_j}. Local
// ancestors are resolved here; the others are requested from rank q (slot
// offset into req[q][1 + s]) and their state will land at particle n + q * bcap
// + s of the next frame's input. cnt[q]: requests to rank q (zeroed after use
// by k_shard_route_fin).
__global__ void k_shard_route(TrackParams P, int rank, int world, const double* __restrict__ bnd,
                              int* __restrict__ req, u32* __restrict__ cnt, i64 bcap) {
  TrackCtl* C = P.ctl;
  const i64 n = P.n;
  const i64 tid = blockIdx.x * (i64)blockDim.x + threadIdx.x, nthr = (i64)gridDim.x * blockDim.x;
  if (!C->do_resample || (C->flags & PCS_FLAG_CAPACITY)) {
    shard_identity(P, C, tid, nthr);
    return;
  }
  const u32 f = C->res_frame;
  bool over = false;
  for (i64 jl = tid; jl < n; jl += nthr) {
    const double p = philox_multinomial_u(P.seed, f, (u64)(P.idx_off + jl));
    int q = 0;
    for (int b = 1; b < world; ++b) q += (bnd[b] <= p) ? 1 : 0;
    if (q == rank) {
      P.anc[jl] = (int)local_search(P.cdf, n, p);
    } else {
      const u32 s = atomicAdd(cnt + q, 1u);
      if ((i64)s < bcap) {
        req[(i64)q * (1 + bcap) + 1 + s] = (int)jl;
        P.anc[jl] = (int)(n + (i64)q * bcap + s);
      } else {
        over = true;
      }
    }
  }
  if (over) set_flag(C, PCS_FLAG_CAPACITY);
}

// request counts into the send buffer (slot 0 of each rank's chunk); sent[q]
// keeps them for the install; cnt is zeroed for the next frame
__global__ void k_shard_route_fin(TrackParams P, int world, int* __restrict__ req,
                                  u32* __restrict__ cnt, u32* __restrict__ sent, i64 bcap) {
  const TrackCtl* C = P.ctl;
  const bool on = C->do_resample && !(C->flags & PCS_FLAG_CAPACITY);
  for (int q = threadIdx.x; q < world; q += blockDim.x) {
    const u32 c = on ? (u32)min((i64)cnt[q], bcap) : 0u;
    req[(i64)q * (1 + bcap)] = (int)c;
    sent[q] = c;
    cnt[q] = 0;
  }
}

// answer the other ranks' requests: state of the local ancestor of each
// requested slot into resp[r][5][bcap]
__global__ void k_shard_serve(TrackParams P, int rank, int world, const int* __restrict__ req_in,
                              float* __restrict__ resp, i64 bcap) {
  const TrackCtl* C = P.ctl;
  if (!C->do_resample || (C->flags & PCS_FLAG_CAPACITY)) return;
  const i64 n = P.n, ld = P.ld;
  const float* cur = (C->k & 1) ? P.buf1 : P.buf0;   // this frame's propagated states
  const u32 f = C->res_frame;
  const i64 total = (i64)world * bcap;
  for (i64 t = blockIdx.x * (i64)blockDim.x + threadIdx.x; t < total; t += (i64)gridDim.x * blockDim.x) {
    const int r = (int)(t / bcap);
    const i64 s = t - (i64)r * bcap;
    const int* chunk = req_in + (i64)r * (1 + bcap);
    if (r == rank || s >= (i64)chunk[0]) continue;
    const i64 j = (i64)r * n + chunk[1 + s];   // the requesting rank's global slot
    const i64 i = local_search(P.cdf, n, philox_multinomial_u(P.seed, f, (u64)j));
    float* o = resp + (i64)r * 5 * bcap;
#pragma unroll
    for (int c = 0; c < 5; ++c) o[c * bcap + s] = cur[c * ld + i];
  }
}

// the answers go to particles n + q * bcap + s (k_shard_route pointed the
// slots at them)
__global__ void k_shard_install(TrackParams P, int rank, int world, const float* __restrict__ resp_in,
                                const u32* __restrict__ sent, i64 bcap) {
  const TrackCtl* C = P.ctl;
  if (!C->do_resample || (C->flags & PCS_FLAG_CAPACITY)) return;
  const i64 n = P.n, ld = P.ld;
  float* cur = (C->k & 1) ? P.buf1 : P.buf0;
  const i64 total = (i64)world * bcap;
  for (i64 t = blockIdx.x * (i64)blockDim.x + threadIdx.x; t < total; t += (i64)gridDim.x * blockDim.x) {
    const int q = (int)(t / bcap);
    const i64 s = t - (i64)q * bcap;
    if (q == rank || s >= (i64)sent[q]) continue;
    const float* in = resp_in + (i64)q * 5 * bcap;
#pragma unroll
    for (int c = 0; c < 5; ++c) cur[c * ld + n + (i64)q * bcap + s] = in[c * bcap + s];
  }
}

}  // namespace pcs
