// pipe_bench.cu -- per-SM throughput of FFMA, FFMA2, FADD2, IMAD, F2FP, FMNMX on this GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/pipe_bench.cu -o scripts/pipe_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float *out, int iters, float seed) {
  float a[16];
  uint64_t b[8];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = seed * (threadIdx.x + i);
#pragma unroll
  for (int i = 0; i < 8; ++i) asm("mov.b64 %0, {%1,%2};" : "=l"(b[i]) : "f"(a[2 * i]), "f"(a[2 * i + 1]));
  const uint64_t c2 = b[0];
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) {  // 2 FFMA
        a[2 * i] = fmaf(a[2 * i], 0.999f, 0.001f);
        a[2 * i + 1] = fmaf(a[2 * i + 1], 0.999f, 0.001f);
      } else if (MODE == 1) {  // 1 FFMA2
        asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(b[i]) : "l"(c2));
      } else if (MODE == 2) {  // 1 FADD2
        asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(b[i]) : "l"(c2));
      } else if (MODE == 3) {  // 2 IMAD (int)
        int u = __float_as_int(a[2 * i]), v = __float_as_int(a[2 * i + 1]);
        asm volatile("mad.lo.s32 %0, %0, 3, %1;" : "+r"(u) : "r"(v));
        asm volatile("mad.lo.s32 %0, %0, 5, %1;" : "+r"(v) : "r"(u));
        a[2 * i] = __int_as_float(u); a[2 * i + 1] = __int_as_float(v);
      } else if (MODE == 4) {  // 1 F2FP (cvt.rn.bf16x2.f32)
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[2 * i]), "f"(a[2 * i + 1]));
        a[2 * i] = __int_as_float(r);
      } else if (MODE == 5) {  // 2 FMNMX
        a[2 * i] = fmaxf(a[2 * i], a[2 * i + 1] * 0.f - 1.f);
        asm volatile("max.f32 %0, %0, %1;" : "+f"(a[2 * i + 1]) : "f"(a[2 * i]));
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) s += __int_as_float((int)b[i]);
  if (s == 12345.f) out[0] = s;
}

int main() {
  float *d;
  cudaMalloc(&d, 4);
  const char *nm[] = {"2x FFMA", "1x FFMA2", "1x FADD2", "2x IMAD", "1x F2FP", "2x FMNMX"};
  for (int mode = 0; mode < 6; ++mode) {
    auto fn = mode == 0 ? k<0> : mode == 1 ? k<1> : mode == 2 ? k<2> : mode == 3 ? k<3> : mode == 4 ? k<4> : k<5>;
    int warps = 16, iters = 4096;
    fn<<<148, warps * 32>>>(d, iters, 1.f);
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    fn<<<148, warps * 32>>>(d, iters, 1.f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double warp_instr_groups = 148.0 * warps * iters * 8;  // each group = one "op" line above per warp
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double cyc = ms * 1e-3 * clk * 1e3;
    printf("%-10s  %.2f groups/clk/SMSP  (%.2f cycles per warp-group per SMSP)\n", nm[mode],
           warp_instr_groups / 148 / 4 / cyc, 148 * 4 * cyc / warp_instr_groups);
  }
  return 0;
}
