// Diagnostic: device time of an (almost) empty single-CTA kernel as a
// function of block size and dynamic shared memory, launched after a
// full-GPU kernel with a large shared-memory footprint (like k_pc_step1).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void big(float* p) {
  extern __shared__ float s[];
  s[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (threadIdx.x == 0) p[blockIdx.x] = s[5];
}
__global__ void tiny(float* p, int nfloat) {
  extern __shared__ float s[];
  __shared__ float st[1024];
  st[threadIdx.x] = 1.0f;
  if ((int)threadIdx.x < nfloat) s[threadIdx.x] = 1.0f;
  __syncthreads();
  if (threadIdx.x == 0) p[0] += st[3] + (nfloat > 3 ? s[3] : 0.f);
}

int main() {
  float* p;
  cudaMalloc(&p, 1 << 20);
  cudaMemset(p, 0, 1 << 20);
  cudaFuncSetAttribute(big, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(tiny, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b, c;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventCreate(&c);
  int blocks[] = {256, 1024};
  int smems[] = {0, 16 * 1024, 64 * 1024, 150 * 1024, 190 * 1024};
  for (int carve = 0; carve < 2; ++carve) {
    if (carve) {
      cudaFuncSetAttribute(big, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      cudaFuncSetAttribute(tiny, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    }
    for (int bs : blocks)
      for (int sm : smems) {
        float tot_ab = 0, tot_bc = 0;
        for (int r = 0; r < 20; ++r) {
          cudaEventRecord(a);
          big<<<148, 512, 198 * 1024>>>(p);
          cudaEventRecord(b);
          tiny<<<1, bs, sm>>>(p, sm / 4);
          cudaEventRecord(c);
          cudaEventSynchronize(c);
          float ab, bc;
          cudaEventElapsedTime(&ab, a, b);
          cudaEventElapsedTime(&bc, b, c);
          if (r >= 5) {
            tot_ab += ab;
            tot_bc += bc;
          }
        }
        printf("carveout_max=%d block=%4d smem=%6d  big=%.2f us  tiny=%.2f us  (%s)\n", carve, bs,
               sm, tot_ab / 15 * 1e3, tot_bc / 15 * 1e3, cudaGetErrorString(cudaGetLastError()));
      }
  }
  return 0;
}
