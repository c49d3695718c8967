// pipe_bench.cu -- per-SM throughput of FFMA, FFMA2, FADD2, IMAD, F2FP, FMNMX, FHADD.BF16,
// MUFU.EX2 and the softmax's per-pair instruction mixes on this GPU.
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
      } else if (MODE == 6) {  // 2 FHADD.BF16 (mixed-precision bf16 + f32 adds)
        const uint32_t pk = __float_as_uint(a[(2 * i + 3) & 15]);
        asm volatile("{ .reg .b16 l, h; mov.b32 {l, h}, %1; add.rn.f32.bf16 %0, l, %0; }" : "+f"(a[2 * i]) : "r"(pk));
        asm volatile("{ .reg .b16 l, h; mov.b32 {l, h}, %1; add.rn.f32.bf16 %0, h, %0; }" : "+f"(a[2 * i + 1]) : "r"(pk));
      } else if (MODE == 7) {  // 2 MUFU.EX2
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[2 * i]));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[2 * i + 1]));
      } else if (MODE == 8) {  // 2 MUFU.EX2 + 2 FHADD (independent)
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[2 * i]));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[2 * i + 1]));
        const uint32_t pk = (uint32_t)b[i];
        float t0 = __int_as_float((int)(b[i] >> 32));
        asm volatile("{ .reg .b16 l, h; mov.b32 {l, h}, %1; add.rn.f32.bf16 %0, l, %0; add.rn.f32.bf16 %0, h, %0; }" : "+f"(t0) : "r"(pk));
        b[i] = (b[i] & 0xffffffffull) | ((uint64_t)__float_as_uint(t0) << 32);
      } else if (MODE == 9) {  // 2 MUFU.EX2 + 1 FADD2 (independent)
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[2 * i]));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[2 * i + 1]));
        asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(b[i]) : "l"(c2));
      } else if (MODE == 10) {  // 2 MUFU.EX2 + 1 FFMA2 + 1 F2FP + 2 FHADD (the softmax pair)
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[2 * i]));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[2 * i + 1]));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(b[i]) : "l"(c2));
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[(2 * i + 5) & 15]), "f"(a[(2 * i + 7) & 15]));
        float t = a[(2 * i + 9) & 15];
        asm volatile("{ .reg .b16 l, h; mov.b32 {l, h}, %1; add.rn.f32.bf16 %0, l, %0; add.rn.f32.bf16 %0, h, %0; }" : "+f"(t) : "r"(r));
        a[(2 * i + 9) & 15] = t;
      } else if (MODE == 11) {  // 2 MUFU.EX2 + 1 FFMA2 + 1 F2FP + 1 FADD2 (fp32 row sum)
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[2 * i]));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[2 * i + 1]));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(b[i]) : "l"(c2));
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[(2 * i + 5) & 15]), "f"(a[(2 * i + 7) & 15]));
        a[(2 * i + 9) & 15] = __int_as_float(r);
        asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(b[(i + 3) & 7]) : "l"(c2));
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
  const char *nm[] = {"2x FFMA", "1x FFMA2", "1x FADD2", "2x IMAD", "1x F2FP", "2x FMNMX", "2x FHADD",
                      "2x MUFU", "2MUFU+2FHADD", "2MUFU+FADD2", "pair:FHADD", "pair:FADD2"};
  void (*fns[])(float *, int, float) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>, k<6>, k<7>, k<8>, k<9>, k<10>, k<11>};
  for (int mode = 0; mode < 12; ++mode) {
    auto fn = fns[mode];
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
