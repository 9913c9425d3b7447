// pcs_bin.cuh — particle-to-cell binning, occupied-bin partition and the
// per-bin dummy reduction (general sort path).
//
// Reference: binning.py:61-67 (cell_indices), :97-112 (_partition: flat id,
// stable argsort, unique/starts/counts), :157-172 (_dummy_states: CoM mean
// via reduceat, weighted CoM, cell-centre placement).
#pragma once
#include "pcs_common.cuh"
#include "pcs_weights.cuh"

namespace pcs {

// flat[i] = iy * n_cols + ix ; idx[i] = i
__global__ void k_cell_keys(const float* __restrict__ s, i64 ld, i64 n, Grid g,
                            u64* __restrict__ flat, int* __restrict__ idx, u32* flags) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    float x = s[i], y = s[ld + i];
    if (!(x == x) || !(y == y)) atomicOr(flags, (u32)PCS_FLAG_NONFINITE);
    i64 ix, iy;
    cell_of(g, x, y, ix, iy);
    flat[i] = (u64)iy * (u64)g.ncols + (u64)ix;
    idx[i] = (int)i;
  }
}

// head flags of the sorted keys -> bin rank per sorted position (via scan)
__global__ void k_run_heads(const u64* __restrict__ sorted, i64 n, int* __restrict__ head) {
  for (i64 p = blockIdx.x * (i64)blockDim.x + threadIdx.x; p < n; p += (i64)gridDim.x * blockDim.x)
    head[p] = (p == 0 || sorted[p] != sorted[p - 1]) ? 1 : 0;
}

// rank (inclusive scan of heads, minus 1) scattered back to particle order
__global__ void k_scatter_bin_of(const int* __restrict__ incl, const int* __restrict__ order, i64 n,
                                 int* __restrict__ bin_of) {
  for (i64 p = blockIdx.x * (i64)blockDim.x + threadIdx.x; p < n; p += (i64)gridDim.x * blockDim.x)
    bin_of[order[p]] = incl[p] - 1;
}

// Exact per-bin sums over sorted members: S_c(b) = sum round(s_c * 2^40);
// weighted: SW_c(b) = sum round(w 2^62) * round(s_c 2^40), SWq(b) = sum round(w 2^62).
// Sorted order keeps bins contiguous, so a warp segments by bin rank and one
// lane per segment issues the (order-free, deterministic) integer atomics.
__global__ void k_bin_sums(const float* __restrict__ s, i64 ld, i64 n, const int* __restrict__ order,
                           const int* __restrict__ bin_of, const float* __restrict__ prior_w,
                           u64* __restrict__ sums /*[6][m][2]*/, i64 m) {
  const int lane = threadIdx.x & 31;
  for (i64 base = (blockIdx.x * (i64)blockDim.x + threadIdx.x) - lane; base < n;
       base += (i64)gridDim.x * blockDim.x) {
    i64 p = base + lane;
    bool valid = p < n;
    int b = -1;
    i128 v[6] = {0, 0, 0, 0, 0, 0};
    if (valid) {
      i64 i = order[p];
      b = bin_of[i];
      i128 wq = prior_w ? f32_to_fixed(prior_w[i], FX_WQ) : (i128)1;
#pragma unroll
      for (int c = 0; c < 5; ++c) v[c] = f32_to_fixed(s[c * ld + i], FX_STATE) * wq;
      v[5] = wq;
    }
    unsigned peers = __match_any_sync(0xffffffffu, b);
    int leader = __ffs(peers) - 1;
    // segmented reduction: leader accumulates peers' values in lane order
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      u64 lo = (u64)v[c], hi = (u64)((u128)v[c] >> 64);
      i128 acc = 0;
      unsigned mset = peers;
      while (mset) {
        int src = __ffs(mset) - 1;
        mset &= mset - 1;
        u64 olo = __shfl_sync(peers, lo, src);
        u64 ohi = __shfl_sync(peers, hi, src);
        acc += (i128)(((u128)ohi << 64) | (u128)olo);
      }
      if (valid && lane == leader) atomic_add_i128(sums + ((i64)c * m + b) * 2, acc);
    }
  }
}

// dummies from the exact sums (CANONICAL):
//   CoM:          d_c = RN32( RN64( RN64(S_c) / count ) * 2^-40 )
//   weighted CoM: d_c = RN32( RN64( RN64(SW_c) / RN64(SWq) ) * 2^-40 )
//   cell centre:  x,y = RN32( origin + (i + 0.5) * cell )   (binning.py:69-71,168-171)
__global__ void k_dummies(const u64* __restrict__ sums, const i64* __restrict__ counts,
                          const u64* __restrict__ unique, i64 m, Grid g, int placement,
                          int weighted, float* __restrict__ d, i64 ldd) {
  for (i64 b = blockIdx.x * (i64)blockDim.x + threadIdx.x; b < m; b += (i64)gridDim.x * blockDim.x) {
    double den = weighted ? i128_to_f64_rn(load_i128(sums + ((i64)5 * m + b) * 2))
                          : (double)counts[b];
#pragma unroll
    for (int c = 0; c < 5; ++c) {
      double num = i128_to_f64_rn(load_i128(sums + ((i64)c * m + b) * 2));
      double mean = scalbn(__ddiv_rn(num, den), -FX_STATE);  // Wq scales cancel when weighted
      d[c * ldd + b] = __double2float_rn(mean);
    }
    if (placement == 1) {
      u64 f = unique[b];
      i64 ix = (i64)(f % (u64)g.ncols), iy = (i64)(f / (u64)g.ncols);
      d[b] = __double2float_rn(__dadd_rn(g.ox, __dmul_rn((double)ix + 0.5, g.lx)));
      d[ldd + b] = __double2float_rn(__dadd_rn(g.oy, __dmul_rn((double)iy + 0.5, g.ly)));
    }
  }
}

// ---- make_dummy (binning.py:129-154): one cell's representative state ----
// float64 members (n, 5) row-major, as the reference. One thread, in the
// reference's summation orders: np.add.reduceat(rows, [0], axis=0) is the
// first row plus numpy's pairwise sum of the remaining rows per column; the
// weight total w.sum() is the pairwise sum of w (blocks of 8 partial sums up
// to 128 elements, recursive halving above); the weighted numerator w @ rows
// is accumulated row by row (BLAS order is implementation-defined; exact for
// exact data).
__device__ double np_pairwise_sum(const double* a, i64 n, i64 stride = 1) {
  // iterative post-order form of numpy's recursive pairwise_sum
  // (PW_BLOCKSIZE 128, 8 partial sums); ops: 0 = sum a range, 1 = add the
  // two most recent results (left + right)
  double vals[64];
  int op_kind[128];
  i64 op_lo[128], op_n[128];
  int top = 0, vp = 0;
  op_kind[top] = 0; op_lo[top] = 0; op_n[top] = n; ++top;
  while (top > 0) {
    --top;
    const int kind = op_kind[top];
    const i64 lo = op_lo[top], m = op_n[top];
    if (kind == 1) {
      const double r = vals[vp - 1], l = vals[vp - 2];
      vp -= 2;
      vals[vp++] = __dadd_rn(l, r);
      continue;
    }
    const double* x = a + lo * stride;
    if (m < 8) {
      double res = -0.0;
      for (i64 i = 0; i < m; ++i) res = __dadd_rn(res, x[i * stride]);
      vals[vp++] = res;
    } else if (m <= 128) {
      double r[8];
      for (int q = 0; q < 8; ++q) r[q] = x[q * stride];
      i64 i;
      for (i = 8; i < m - (m % 8); i += 8)
        for (int q = 0; q < 8; ++q) r[q] = __dadd_rn(r[q], x[(i + q) * stride]);
      double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                             __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
      for (; i < m; ++i) res = __dadd_rn(res, x[i * stride]);
      vals[vp++] = res;
    } else {
      i64 n2 = m / 2;
      n2 -= n2 % 8;
      op_kind[top] = 1; op_lo[top] = 0; op_n[top] = 0; ++top;            // then combine
      op_kind[top] = 0; op_lo[top] = lo + n2; op_n[top] = m - n2; ++top;  // right second
      op_kind[top] = 0; op_lo[top] = lo; op_n[top] = n2; ++top;           // left first
    }
  }
  return vals[0];
}

__global__ void k_make_dummy(const double* __restrict__ rows, i64 n, const double* __restrict__ w,
                             int placement, double x_lo, double x_hi, double y_lo, double y_hi,
                             double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double mean[5];
  if (w) {
    double num[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (i64 i = 0; i < n; ++i)
      for (int c = 0; c < 5; ++c) num[c] = __dadd_rn(num[c], __dmul_rn(w[i], rows[i * 5 + c]));
    const double den = np_pairwise_sum(w, n);
    for (int c = 0; c < 5; ++c) mean[c] = __ddiv_rn(num[c], den);
  } else {
    for (int c = 0; c < 5; ++c) {
      const double acc = (n == 1) ? rows[c] : __dadd_rn(rows[c], np_pairwise_sum(rows + 5 + c, n - 1, 5));
      mean[c] = __ddiv_rn(acc, (double)n);
    }
  }
  if (placement == 1) {   // cell centre (binning.py:150-153)
    mean[0] = __ddiv_rn(__dadd_rn(x_lo, x_hi), 2.0);
    mean[1] = __ddiv_rn(__dadd_rn(y_lo, y_hi), 2.0);
  }
  for (int c = 0; c < 5; ++c) out[c] = mean[c];
}

}  // namespace pcs
