// exp_bench.cu -- MUFU.EX2 vs FMA-pipe polynomial exp2 throughput on this GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/exp_bench.cu -o scripts/exp_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float poly(float x) {
  x = fmaxf(x, -127.f);
  float t = x + 12582912.0f;
  float r = t - 12582912.0f;
  float f = x - r;
  float p = fmaf(f, 0.055008627f, 0.24221043f);
  p = fmaf(p, f, 0.69328302f);
  p = fmaf(p, f, 1.0f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

template <int MODE>
__global__ void k(float *out, int iters, float seed) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = seed * (threadIdx.x + i) * 1e-9f - 0.5f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float v = MODE == 0 ? ex2(a[i]) : poly(a[i]);
      a[i] = v * -0.999f;  // keep values bounded and dependent (1 FMUL per exp)
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 12345.f) out[0] = s;
}

int main() {
  float *d;
  cudaMalloc(&d, 4);
  for (int mode = 0; mode < 2; ++mode) {
    for (int warps : {4, 8, 16}) {
      auto fn = mode == 0 ? k<0> : k<1>;
      int iters = 2048;
      fn<<<148, warps * 32>>>(d, iters, 1.f);
      cudaDeviceSynchronize();
      cudaEvent_t a, b;
      cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      fn<<<148, warps * 32>>>(d, iters, 1.f);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double n = 148.0 * warps * 32 * iters * 16;
      int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
      double per_sm_clk = n / 148 / (ms * 1e-3 * clk * 1e3);
      printf("%s warps/SM=%2d  %.2f Gexp/s  ~%.1f exp/clk/SM (at %d MHz)\n", mode ? "poly " : "MUFU ", warps,
             n / (ms * 1e-3) / 1e9, per_sm_clk, clk / 1000);
    }
  }
  return 0;
}
