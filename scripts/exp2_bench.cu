// exp2_bench.cu -- MUFU.EX2 throughput: f32 vs f16x2 vs bf16x2 inputs (results per clk per SM).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/exp2_bench.cu -o scripts/exp2_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float *out, int iters, float seed) {
  uint32_t a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    float f = -seed * (threadIdx.x + i) * 1e-6f;
    a[i] = MODE == 0 ? __float_as_uint(f) : 0xbc00bc00u;  // -1.0 (f16x2) / tiny neg (bf16x2)
    if (MODE == 2) a[i] = 0xbf80bf80u;                    // -1.0 bf16x2
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) {
        float y;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(__uint_as_float(a[i])));
        a[i] = __float_as_uint(-y);
      } else if (MODE == 1) {
        uint32_t y;
        asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(a[i]));
        a[i] = y | 0x80008000u;
      } else {
        uint32_t y;
        asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(a[i]));
        a[i] = y | 0x80008000u;
      }
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s ^= a[i];
  if (s == 12345u) out[0] = s;
}

int main() {
  float *d;
  cudaMalloc(&d, 4);
  const char *nm[] = {"f32   ", "f16x2 ", "bf16x2"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int warps : {4, 8, 16}) {
      auto fn = mode == 0 ? k<0> : mode == 1 ? k<1> : k<2>;
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
      double instr = 148.0 * warps * 32 * iters * 16;  // thread-instructions
      int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
      double per_sm_clk = instr / 148 / (ms * 1e-3 * clk * 1e3);
      printf("%s warps/SM=%2d  %.1f thread-instr/clk/SM -> %.1f exp/clk/SM\n", nm[mode], warps, per_sm_clk,
             per_sm_clk * (mode ? 2 : 1));
    }
  }
  return 0;
}
