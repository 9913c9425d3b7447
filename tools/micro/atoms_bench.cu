// Shared-memory 32-bit atomic throughput on B200: NATOM adds per "particle"
// into [NATOM][1024] u32 accumulators, cell drawn from a distribution of
// `ncell` effective cells (mode 0 uniform over ncell, mode 1 gaussian-ish)
#include <cstdio>
#include <cuda_runtime.h>
template <int NATOM, bool RED>
__global__ void __launch_bounds__(512, 2) k(unsigned* out, int iters, int ncell, int mode) {
  extern __shared__ unsigned accraw[];
  unsigned (*acc)[1024] = reinterpret_cast<unsigned (*)[1024]>(accraw);
  for (int i = threadIdx.x; i < NATOM * 1024; i += 512) (&acc[0][0])[i] = 0;
  __syncthreads();
  unsigned s = blockIdx.x * 7919u + threadIdx.x * 104729u + 1;
  unsigned sum = 0;
  for (int it = 0; it < iters; ++it) {
    s = s * 1664525u + 1013904223u;
    unsigned q;
    if (mode == 0) q = (s >> 8) % ncell;
    else { unsigned a = (s >> 4) & 0xFF, b = (s >> 12) & 0xFF, c = (s >> 20) & 0xFF; q = ((a + b + c) * ncell / 765u) % ncell; }
#pragma unroll
    for (int c2 = 0; c2 < NATOM; ++c2) {
      if (RED) atomicAdd(&acc[c2][q], s & (0x3FFFFu >> c2));
      else sum += atomicAdd(&acc[c2][q], s & (0x3FFFFu >> c2));
    }
  }
  __syncthreads();
  unsigned v = sum;
  for (int i = threadIdx.x; i < NATOM * 1024; i += 512) v += (&acc[0][0])[i];
  out[blockIdx.x * 512 + threadIdx.x] = v;
}
template <int NATOM, bool RED>
void run(unsigned* d, int ncell, int mode) {
  int iters = 4096;
  int grid = 148 * 2;
  cudaFuncSetAttribute(k<NATOM, RED>, cudaFuncAttributeMaxDynamicSharedMemorySize, NATOM*4096);
  k<NATOM, RED><<<grid, 512, NATOM*4096>>>(d, 16, ncell, mode);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<NATOM, RED><<<grid, 512, NATOM*4096>>>(d, iters, ncell, mode);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double parts = (double)grid * 512 * iters;
  printf("NATOM=%2d red=%d ncell=%4d mode=%d: %.3f ms, %.3f ns/Mparticle-equiv -> %.2f Gparticles/s, %.2f cyc/atom-lane/SM\n",
         NATOM, RED, ncell, mode, ms, ms * 1e6 / parts * 1e6, parts / ms / 1e6,
         (ms * 1e-3 * 1.965e9) / (parts * NATOM / 148.0));
}
int main() {
  unsigned* d; cudaMalloc(&d, 148 * 2 * 512 * 4);
  for (int mode = 0; mode < 2; ++mode)
    for (int nc : {32, 256, 1024}) {
      run<1, true>(d, nc, mode);
      run<12, true>(d, nc, mode);
      run<16, true>(d, nc, mode);
      run<16, false>(d, nc, mode);
    }
  return 0;
}
