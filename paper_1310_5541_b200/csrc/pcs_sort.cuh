// pcs_sort.cuh — stable LSD radix sort of (cell key, particle index) pairs
// and the run-length partition of the per-step API (binning.py:97-112:
// flat id, stable argsort, unique / starts / counts).
//
// Keys are the flat cell ids (up to 64 bits: acceptance #1 grids have
// ~4e13 cells); only the bits of the largest id are sorted, 8 per pass.
// One pass = three launches over tiles of RS8_TILE pairs:
//   k_radix_hist     digit histogram of every tile  -> hist[digit][tile]
//   scan_excl_i32    exclusive scan of hist (digit-major), i.e. every
//                    (digit, tile)'s first output position
//   k_radix_scatter  stable rank of each pair among the tile's pairs with
//                    the same digit, then scatter keys and indices
// Stable ranks without per-thread histograms: warp w handles tile
// positions [w*512, (w+1)*512) in batches of 32 consecutive pairs (lane =
// position, coalesced loads); __match_any_sync groups a batch's equal
// digits, a pair's rank is the running count of its digit in the warp
// (shared memory) plus the number of equal-digit lanes below it; the
// per-warp counts are then scanned over the warps per digit.
#pragma once
#include "pcs_common.cuh"

namespace pcs {

constexpr int RS8_THREADS = 256;
constexpr int RS8_WARPS = RS8_THREADS / 32;
constexpr int RS8_BATCHES = 16;                            // batches of 32 per warp
constexpr int RS8_TILE = RS8_THREADS * RS8_BATCHES;       // 4096 pairs per tile

__global__ void __launch_bounds__(RS8_THREADS) k_radix_hist(const u64* __restrict__ keys, i64 n,
                                                           int shift, i64 ntiles,
                                                           int* __restrict__ hist) {
  __shared__ int cnt[256];
  const i64 tile = blockIdx.x;
  cnt[threadIdx.x] = 0;
  __syncthreads();
  const i64 t0 = tile * RS8_TILE;
  for (int k = threadIdx.x; k < RS8_TILE; k += RS8_THREADS) {
    const i64 p = t0 + k;
    if (p < n) atomicAdd(&cnt[(int)((keys[p] >> shift) & 0xFFull)], 1);
  }
  __syncthreads();
  hist[(i64)threadIdx.x * ntiles + tile] = cnt[threadIdx.x];
}

__global__ void __launch_bounds__(RS8_THREADS) k_radix_scatter(
    const u64* __restrict__ kin, const int* __restrict__ vin, u64* __restrict__ kout,
    int* __restrict__ vout, i64 n, int shift, i64 ntiles, const int* __restrict__ offs) {
  __shared__ int wcnt[RS8_WARPS][256];   // running / then exclusive per-warp digit counts
  __shared__ int gofs[256];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const i64 tile = blockIdx.x;
  for (int d = lane; d < 256; d += 32) wcnt[w][d] = 0;
  gofs[threadIdx.x] = offs[(i64)threadIdx.x * ntiles + tile];
  __syncwarp();
  const i64 base = tile * RS8_TILE + (i64)w * (32 * RS8_BATCHES);
  const unsigned lt = (1u << lane) - 1u;
  int local[RS8_BATCHES];
#pragma unroll
  for (int b = 0; b < RS8_BATCHES; ++b) {
    const i64 p = base + b * 32 + lane;
    const int d = (p < n) ? (int)((kin[p] >> shift) & 0xFFull) : 256;   // 256: no pair
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const int before = (d < 256) ? wcnt[w][d] : 0;
    local[b] = before + __popc(peers & lt);
    __syncwarp();
    if (d < 256 && lane == 31 - __clz(peers)) wcnt[w][d] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  {   // exclusive scan over the warps, per digit (thread = digit)
    const int d = threadIdx.x;
    int run = 0;
#pragma unroll
    for (int ww = 0; ww < RS8_WARPS; ++ww) {
      const int c = wcnt[ww][d];
      wcnt[ww][d] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int b = 0; b < RS8_BATCHES; ++b) {
    const i64 p = base + b * 32 + lane;
    if (p < n) {
      const u64 key = kin[p];
      const int d = (int)((key >> shift) & 0xFFull);
      const i64 dst = (i64)gofs[d] + wcnt[w][d] + local[b];
      kout[dst] = key;
      vout[dst] = vin[p];
    }
  }
}

// ---- exclusive scan of int32 (block partials, recursive on the totals) ----
constexpr int SC_THREADS = 512;
constexpr int SC_ITEMS = 4;
constexpr int SC_BLOCK = SC_THREADS * SC_ITEMS;   // 2048

// in-place exclusive scan of each block of SC_BLOCK items; block totals out
__global__ void __launch_bounds__(SC_THREADS) k_scan_blocks(int* __restrict__ a, i64 n,
                                                           int* __restrict__ totals) {
  __shared__ int wsum[SC_THREADS / 32];
  const i64 b0 = (i64)blockIdx.x * SC_BLOCK + (i64)threadIdx.x * SC_ITEMS;
  int v[SC_ITEMS];
  int s = 0;
#pragma unroll
  for (int q = 0; q < SC_ITEMS; ++q) {
    v[q] = (b0 + q < n) ? a[b0 + q] : 0;
    s += v[q];
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int inc = s;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int o = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += o;
  }
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  int woff = 0, tot = 0;
#pragma unroll
  for (int ww = 0; ww < SC_THREADS / 32; ++ww) {
    if (ww < w) woff += wsum[ww];
    tot += wsum[ww];
  }
  int run = woff + inc - s;
#pragma unroll
  for (int q = 0; q < SC_ITEMS; ++q) {
    if (b0 + q < n) a[b0 + q] = run;
    run += v[q];
  }
  if (threadIdx.x == 0) totals[blockIdx.x] = tot;
}

__global__ void k_scan_add(int* __restrict__ a, i64 n, const int* __restrict__ offs) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    a[i] += offs[i / SC_BLOCK];
}

// run heads of sorted keys: head[p] = 1 where a new key starts
__global__ void k_key_heads(const u64* __restrict__ sorted, i64 n, int* __restrict__ head) {
  for (i64 p = blockIdx.x * (i64)blockDim.x + threadIdx.x; p < n; p += (i64)gridDim.x * blockDim.x)
    head[p] = (p == 0 || sorted[p] != sorted[p - 1]) ? 1 : 0;
}

// from the exclusive scan of the heads (rank of each run): unique keys,
// run starts, bin of every particle; counts from consecutive starts
__global__ void k_runs(const u64* __restrict__ sorted, const int* __restrict__ order, i64 n,
                       const int* __restrict__ rank_excl, u64* __restrict__ unique,
                       i64* __restrict__ starts, int* __restrict__ bin_of) {
  for (i64 p = blockIdx.x * (i64)blockDim.x + threadIdx.x; p < n; p += (i64)gridDim.x * blockDim.x) {
    const bool head = (p == 0 || sorted[p] != sorted[p - 1]);
    const int b = rank_excl[p] + (head ? 0 : -1);   // exclusive scan: head p has rank_excl = b
    if (head) {
      unique[b] = sorted[p];
      starts[b] = p;
    }
    bin_of[order[p]] = b;
  }
}

__global__ void k_run_counts(const i64* __restrict__ starts, i64 m, i64 n, i64* __restrict__ counts) {
  for (i64 b = blockIdx.x * (i64)blockDim.x + threadIdx.x; b < m; b += (i64)gridDim.x * blockDim.x)
    counts[b] = ((b + 1 < m) ? starts[b + 1] : n) - starts[b];
}

}  // namespace pcs
