// accuracy of lg2.approx.ftz.f32 on u = RN(1 + t) against log2(1 + t) (float64)
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
__global__ void k(const float* t, float* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float u = 1.0f + t[i];
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(u));
  out[i] = y;
}
int main() {
  const int n = 1 << 22;
  float* h = (float*)malloc(n * 4);
  float* r = (float*)malloc(n * 4);
  for (int i = 0; i < n; ++i) h[i] = (float)std::exp(std::log(1e-7) + (std::log(8.0) - std::log(1e-7)) * (i + 0.5) / n);
  float *dt, *dy;
  cudaMalloc(&dt, n * 4); cudaMalloc(&dy, n * 4);
  cudaMemcpy(dt, h, n * 4, cudaMemcpyHostToDevice);
  k<<<n / 256, 256>>>(dt, dy, n);
  cudaMemcpy(r, dy, n * 4, cudaMemcpyDeviceToHost);
  // error of log(u) from MUFU vs exact log(u) (u = RN(1+t)), in absolute and relative terms, per decade of t
  double lo = 1e-7;
  while (lo < 8) {
    double hi = lo * 10, maxabs = 0, maxrel = 0, sum = 0; int c = 0;
    for (int i = 0; i < n; ++i) {
      if (h[i] < lo || h[i] >= hi) continue;
      float u = 1.0f + h[i];
      double ex = std::log2((double)u);
      double e = (double)r[i] - ex;
      maxabs = std::fmax(maxabs, std::fabs(e));
      if (ex != 0) maxrel = std::fmax(maxrel, std::fabs(e / ex));
      sum += e; ++c;
    }
    printf("t in [%.0e, %.0e): max abs err %.3e (2^%.1f), max rel %.3e, mean %.3e, n %d\n", lo, hi, maxabs, std::log2(maxabs + 1e-300), maxrel, sum / c, c);
    lo = hi;
  }
  return 0;
}
