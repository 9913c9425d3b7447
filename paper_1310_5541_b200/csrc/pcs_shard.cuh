// pcs_shard.cuh — particle-sharded giant filter (config 5) helpers.
//
// Each rank holds a contiguous global index range of particles. Per frame:
//   k_pc_step1 (local, Philox on global indices) -> local exact cell sums
//   k_shard_bbox         local occupied-cell bounding box  (all-reduce MIN/MAX)
//   k_shard_export       window cells -> 16 int64 limbs per cell, table zeroed
//   NCCL all-reduce SUM  (limbs: exact, associative -> P-invariant)
//   k_shard_import       global sums back into the table + occupied list
//   k_pc_bins            identical on every rank (same inputs, same code)
//   k_scan_emit mode 1   rank-local exact prefix; rank totals all-gathered
//   k_scan_emit mode 2   global slots for this rank's particles
//   NCCL all-to-all      resampled states to the ranks owning their slots
// The int128 per-cell sums are carried as three 42-bit limbs so an int64
// all-reduce over up to 2^21 ranks cannot overflow and the total is exact.
#pragma once
#include "pcs_common.cuh"
#include "pcs_fused.cuh"

namespace pcs {

constexpr int LIMBS_PER_CELL = 16;   // count + 5 components x 3 limbs

__global__ void k_shard_bbox(TrackParams P, i64* out /* ix0, ix1, iy0, iy1, n_occ */) {
  __shared__ long long s[4];
  TrackCtl* C = P.ctl;
  const u32 m = C->n_occ;
  if (threadIdx.x == 0) {
    s[0] = LLONG_MAX;
    s[1] = LLONG_MIN;
    s[2] = LLONG_MAX;
    s[3] = LLONG_MIN;
  }
  __syncthreads();
  const u32 mm = min(m, (u32)MAXM);
  for (u32 b = threadIdx.x; b < mm; b += blockDim.x) {
    u32 cell = P.occ[b];
    long long ix = (long long)cell % P.grid.ncols, iy = (long long)cell / P.grid.ncols;
    atomicMin(&s[0], ix);
    atomicMax(&s[1], ix);
    atomicMin(&s[2], iy);
    atomicMax(&s[3], iy);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 0; q < 4; ++q) out[q] = s[q];
    out[4] = m;
    if (m > (u32)MAXM) set_flag(C, PCS_FLAG_CAPACITY);
  }
}

__global__ void k_shard_export(TrackParams P, i64 x0, i64 y0, i64 nx, i64 ny, i64* __restrict__ limbs) {
  const i64 W = nx * ny;
  const u64 M42 = (1ull << 42) - 1ull;
  if (blockIdx.x == 0 && threadIdx.x == 0) P.ctl->n_occ = 0;   // import rebuilds the list
  for (i64 q = blockIdx.x * (i64)blockDim.x + threadIdx.x; q < W; q += (i64)gridDim.x * blockDim.x) {
    i64 ix = x0 + q % nx, iy = y0 + q / nx;
    i64* L = limbs + q * LIMBS_PER_CELL;
    u32 flat = (u32)(iy * P.grid.ncols + ix);
    u32 cnt = P.tab_cnt[flat];
    L[0] = cnt;
    for (int c = 0; c < 5; ++c) {
      i128 v = 0;
      if (cnt) {
        u64* p = P.tab_sum + ((i64)c * P.G + flat) * 2;
        v = load_i128(p);
        p[0] = 0;
        p[1] = 0;
      }
      L[1 + 3 * c] = (i64)((u64)v & M42);
      L[2 + 3 * c] = (i64)((u64)(v >> 42) & M42);
      L[3 + 3 * c] = (i64)(v >> 84);   // arithmetic shift keeps the sign
    }
    if (cnt) P.tab_cnt[flat] = 0;
  }
}

__global__ void k_shard_import(TrackParams P, i64 x0, i64 y0, i64 nx, i64 ny,
                               const i64* __restrict__ limbs) {
  const i64 W = nx * ny;
  TrackCtl* C = P.ctl;
  for (i64 q = blockIdx.x * (i64)blockDim.x + threadIdx.x; q < W; q += (i64)gridDim.x * blockDim.x) {
    const i64* L = limbs + q * LIMBS_PER_CELL;
    i64 cnt = L[0];
    if (!cnt) continue;
    i64 ix = x0 + q % nx, iy = y0 + q / nx;
    u32 flat = (u32)(iy * P.grid.ncols + ix);
    P.tab_cnt[flat] = (u32)cnt;
    for (int c = 0; c < 5; ++c) {
      i128 v = (i128)L[1 + 3 * c] + ((i128)L[2 + 3 * c] << 42) + ((i128)L[3 + 3 * c] << 84);
      u64* p = P.tab_sum + ((i64)c * P.G + flat) * 2;
      p[0] = (u64)v;
      p[1] = (u64)((u128)v >> 64);
    }
    u32 idx = atomicAdd(&C->n_occ, 1u);
    if (idx < (u32)MAXM) P.occ[idx] = flat;
  }
}

// out[c*count + q] = in[c*ld + anc[q]]
__global__ void k_shard_gather(const float* __restrict__ sin, i64 ld, const int* __restrict__ anc,
                               i64 count, float* __restrict__ out) {
  for (i64 q = blockIdx.x * (i64)blockDim.x + threadIdx.x; q < count; q += (i64)gridDim.x * blockDim.x) {
    i64 src = anc[q];
#pragma unroll
    for (int c = 0; c < 5; ++c) out[c * count + q] = __ldg(sin + c * ld + src);
  }
}

__global__ void k_shard_set_prefix(TrackCtl* C, u64 lo, u64 hi) {
  C->rank_prefix[0] = lo;
  C->rank_prefix[1] = hi;
}

}  // namespace pcs
