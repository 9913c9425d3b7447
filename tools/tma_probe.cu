// Diagnostic: TMA 3D tile load of a 64x16 float box with the tensor map as a
// __grid_constant__ parameter vs in global memory.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <bool GLOBAL_MAP>
__global__ void k(const __grid_constant__ CUtensorMap pmap, const CUtensorMap* gmap, float* out,
                  int x0, int y0) {
  __shared__ __align__(128) float buf[64 * 16];
  __shared__ __align__(8) unsigned long long bar;
  const void* m = GLOBAL_MAP ? (const void*)gmap : (const void*)&pmap;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)),
                 "r"(64 * 16 * 4) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(sa(buf)), "l"(m), "r"(x0), "r"(y0), "r"(0),
        "r"(sa(&bar)) : "memory");
  }
  __syncthreads();
  asm volatile(
      "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
      "@!p bra W_%=;\n\t}" ::"r"(sa(&bar)) : "memory");
  for (int i = threadIdx.x; i < 64 * 16; i += blockDim.x) out[i] = buf[i];
}

// bins-kernel-like: static smem + 226 KB dynamic, boxes at offset 98304
__global__ void k2(const CUtensorMap* gmap, float* out, int x0, int y0, int nb) {
  __shared__ long long s_max;
  __shared__ int s_box[4];
  extern __shared__ __align__(128) unsigned char raw[];
  float* buf = reinterpret_cast<float*>(raw + 98304);
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(raw + 226816);
  if (threadIdx.x == 0) { s_max = 0; s_box[0] = 0; }
  if (threadIdx.x == 0) {
    out[2048] = (float)(sa(buf) & 127);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bar)),
                 "r"(nb * 64 * 16 * 4) : "memory");
    for (int j = 0; j < nb; ++j)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
          "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(sa(buf + j * 1024)), "l"(gmap), "r"(x0),
          "r"(y0 + 16 * j), "r"(0), "r"(sa(bar)) : "memory");
  }
  __syncthreads();
  asm volatile(
      "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
      "@!p bra W_%=;\n\t}" ::"r"(sa(bar)) : "memory");
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) out[i] = buf[i];
}

int main() {
  const int W = 64, H = 64;
  float* f;
  cudaMalloc(&f, W * H * 4);
  float h[W * H];
  for (int i = 0; i < W * H; ++i) h[i] = (float)i;
  cudaMemcpy(f, h, sizeof(h), cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap m;
  cuuint64_t dims[3] = {W, H, 1};
  cuuint64_t str[2] = {W * 4, W * H * 4};
  cuuint32_t box[3] = {64, 16, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, f, dims, str, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  CUtensorMap* g;
  cudaMalloc(&g, sizeof(m));
  cudaMemcpy(g, &m, sizeof(m), cudaMemcpyHostToDevice);
  float* out;
  cudaMalloc(&out, 64 * 16 * 4);
  float ho[64 * 16];
  k<false><<<1, 128>>>(m, g, out, 0, 8);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(ho, out, sizeof(ho), cudaMemcpyDeviceToHost);
  printf("param map: %s  out[0]=%g (want %d) out[65]=%g (want %d)\n", cudaGetErrorString(e), ho[0],
         8 * 64, ho[65], 9 * 64 + 1);
  if (e == cudaSuccess) {
    k<true><<<1, 128>>>(m, g, out, 0, 8);
    e = cudaDeviceSynchronize();
    cudaMemcpy(ho, out, sizeof(ho), cudaMemcpyDeviceToHost);
    printf("global map: %s  out[0]=%g out[65]=%g\n", cudaGetErrorString(e), ho[0], ho[65]);
  }
  cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, 226824);
  float* out2;
  cudaMalloc(&out2, 2049 * 4);
  float ho2[2049];
  int xs = getenv("X0") ? atoi(getenv("X0")) : 0;
  k2<<<1, 512, 226824>>>(g, out2, xs, 8, 2);
  e = cudaDeviceSynchronize();
  cudaMemcpy(ho2, out2, sizeof(ho2), cudaMemcpyDeviceToHost);
  printf("k2 (bins-like): %s  align=%g out[0]=%g (want %d) out[1100]=%g (want %d)\n", 
         cudaGetErrorString(e), ho2[2048], ho2[0], 8 * 64 + xs, ho2[1100], (8 + 17) * 64 + xs + 12);
  return 0;
}
