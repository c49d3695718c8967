// softmax_bench.cu -- cycles per 128-column row block of the softmax exp phase in
// isolation (no TMEM / MMA), for instruction-mix experiments.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/softmax_bench.cu -o scripts/softmax_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t f2pack(float lo, float hi) {
  uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r;
}
__device__ __forceinline__ void f2unpack(uint64_t v, float &lo, float &hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t u2pack(uint32_t lo, uint32_t hi) {
  uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi)); return r;
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t r; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t r; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r;
}
__device__ __forceinline__ float max3(float a, float b, float c) {
  float r; asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c)); return r;
}
__device__ __forceinline__ float ex2(float x) {
  float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  uint32_t r; asm("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(lo), "f"(hi)); return r;
}
__device__ __forceinline__ int lea23(int a, int b) {
  int r; asm("{\n\t.reg .b32 t;\n\tshl.b32 t, %1, 23;\n\tadd.s32 %0, t, %2;\n\t}" : "=r"(r) : "r"(a), "r"(b)); return r;
}
// degree DEG (2 or 3) polynomial exp2 for a pair
template <int DEG>
__device__ __forceinline__ void exp2_poly2(float x0, float x1, float &y0, float &y1) {
  constexpr float kMagic = 12582912.0f;
  x0 = fmaxf(x0, -127.f);
  x1 = fmaxf(x1, -127.f);
  const uint64_t x = f2pack(x0, x1);
  const uint64_t t = fadd2(x, f2pack(kMagic, kMagic));
  const uint64_t r = fadd2(t, f2pack(-kMagic, -kMagic));
  uint64_t f = ffma2(r, f2pack(-1.f, -1.f), x);
  uint64_t pp;
  if (DEG == 3) {
    pp = ffma2(f, f2pack(0.055008627f, 0.055008627f), f2pack(0.24221043f, 0.24221043f));
    pp = ffma2(pp, f, f2pack(0.69328302f, 0.69328302f));
    pp = ffma2(pp, f, f2pack(1.0f, 1.0f));
  } else {
    pp = ffma2(f, f2pack(0.2402265f, 0.2402265f), f2pack(0.6931472f, 0.6931472f));
    pp = ffma2(pp, f, f2pack(1.0f, 1.0f));
  }
  float p0, p1, t0, t1;
  f2unpack(pp, p0, p1);
  f2unpack(t, t0, t1);
  y0 = __int_as_float(lea23(__float_as_int(t0), __float_as_int(p0)));
  y1 = __int_as_float(lea23(__float_as_int(t1), __float_as_int(p1)));
}

// MODE bits: poly mask in bits 0-7; bit 8: degree 2; bit 9: skip max; bit 10: skip rowsum
template <int MODE>
__global__ void __launch_bounds__(256, 1) k(const float *in, uint32_t *out, int iters, long long *cyc) {
  __shared__ uint4 sp[256 * 8];
  const int tid = threadIdx.x;
  uint32_t s[128];
#pragma unroll
  for (int i = 0; i < 128; ++i) s[i] = __float_as_uint(in[(i * 37 + tid) & 1023]);
  float l_run = 0.f, m_run = 0.f;
  const float sc = 0.1275f;
  const uint32_t prow = (uint32_t)__cvta_generic_to_shared(sp) + (tid % 128) * 128;
  const int psw = tid & 7;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float mx = -INFINITY;
    if (!(MODE & 512)) {
      float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
      for (int e = 0; e < 128; e += 8) {
        mx0 = max3(mx0, __uint_as_float(s[e]), __uint_as_float(s[e + 1]));
        mx1 = max3(mx1, __uint_as_float(s[e + 2]), __uint_as_float(s[e + 3]));
        mx2 = max3(mx2, __uint_as_float(s[e + 4]), __uint_as_float(s[e + 5]));
        mx3 = max3(mx3, __uint_as_float(s[e + 6]), __uint_as_float(s[e + 7]));
      }
      mx = max3(mx0, mx1, fmaxf(mx2, mx3));
    }
    const float ref = fmaxf(m_run, mx * sc);
    const uint64_t sc2 = f2pack(sc, sc);
    const uint64_t nref2 = f2pack(-ref, -ref);
    uint64_t l2a = 0, l2b = 0;
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      uint32_t pk[32];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
#pragma unroll
        for (int e = 0; e < 16; e += 2) {
          const int col = hh * 64 + c * 16 + e;
          const uint64_t xx = ffma2(u2pack(s[col], s[col + 1]), sc2, nref2);
          float x0, x1, p0, p1;
          f2unpack(xx, x0, x1);
          if (((MODE & 255) >> ((col >> 1) & 7)) & 1) {
            if (MODE & 256) exp2_poly2<2>(x0, x1, p0, p1); else exp2_poly2<3>(x0, x1, p0, p1);
          } else {
            p0 = ex2(x0);
            p1 = ex2(x1);
          }
          if (!(MODE & 1024)) {
            if (e & 2) l2b = fadd2(l2b, f2pack(p0, p1));
            else l2a = fadd2(l2a, f2pack(p0, p1));
          }
          pk[c * 8 + e / 2] = pack_bf16(p0, p1);
        }
      }
#pragma unroll
      for (int c = 0; c < 8; ++c)
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(prow + ((c ^ psw) << 4)), "r"(pk[4 * c]),
                     "r"(pk[4 * c + 1]), "r"(pk[4 * c + 2]), "r"(pk[4 * c + 3]) : "memory");
    }
    const uint64_t l2 = fadd2(l2a, l2b);
    float a0, a1;
    f2unpack(l2, a0, a1);
    l_run += a0 + a1;
    m_run = ref * 0.5f;
    // perturb s so the compiler cannot hoist
#pragma unroll
    for (int i = 0; i < 128; i += 16) s[i] ^= (uint32_t)it & 1u;
  }
  long long t1 = clock64();
  if (tid % 32 == 0) cyc[blockIdx.x * 8 + tid / 32] = t1 - t0;
  if (l_run == 1.2345f) out[0] = 1;
}

template <int MODE>
void run(const char *name, int warps, const float *in, uint32_t *out, long long *cyc) {
  const int iters = 512;
  k<MODE><<<148, warps * 32>>>(in, out, 8, cyc);
  cudaDeviceSynchronize();
  k<MODE><<<148, warps * 32>>>(in, out, iters, cyc);
  cudaDeviceSynchronize();
  long long h[148 * 8];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int b = 0; b < 148; ++b)
    for (int w = 0; w < warps; ++w) avg += h[b * 8 + w];
  avg /= 148 * warps;
  printf("%-28s warps/SMSP=%d  %7.0f cycles per warp-block  (%7.0f per SMSP-block)\n", name, warps / 4, avg / iters,
         avg / iters / (warps / 4));
}

int main() {
  float *in; uint32_t *out; long long *cyc;
  cudaMalloc(&in, 4096 * 4); cudaMalloc(&out, 4); cudaMalloc(&cyc, 148 * 8 * 8);
  float h[1024];
  for (int i = 0; i < 1024; ++i) h[i] = (float)((i * 7919) % 1000) / 100.f - 5.f;
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int w : {4, 8}) {
    run<0x25>("poly 3/8 deg3", w, in, out, cyc);
    run<0x00>("all MUFU", w, in, out, cyc);
    run<0x11>("poly 1/4 deg3", w, in, out, cyc);
    run<0x55>("poly 1/2 deg3", w, in, out, cyc);
    run<0x125>("poly 3/8 deg2", w, in, out, cyc);
    run<0x155>("poly 1/2 deg2", w, in, out, cyc);
    run<0x225>("poly 3/8 deg3 nomax", w, in, out, cyc);
    run<0x425>("poly 3/8 deg3 nosum", w, in, out, cyc);
    run<0x625>("poly 3/8 nomax nosum", w, in, out, cyc);
  }
  return 0;
}
