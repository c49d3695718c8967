// kernels.cu -- sm_100a kernels of the TriangleMix prefill-attention hot path.
//
//  attn_kernel<D>   persistent, warp-specialised flash attention over the static
//                   item schedule (schedule.h): STREAM items (sink + sliding-window
//                   band, Algorithm 1 "upper part"), LASTQ split-K items
//                   (Algorithm 1 "last rows") and DENSE items (causal,
//                   P:L257-261).  QK^T and PV are tcgen05 MMAs accumulating in TMEM,
//                   K/V blocks arrive through a multi-stage TMA ring, the online softmax
//                   (Algorithm 1's flash_attn, P:L610/L618/L634) runs one query row per
//                   thread straight out of TMEM.
//  merge_kernel<D>  LSE merge of the split-K partials (merge_output).
//
// CTA layout (384 threads, 1 CTA per SM):
//   warp 0      TMA producer (one elected lane)
//   warp 1      MMA issuer  (one elected lane)
//   warp 2      TMEM allocator
//   warp 3      idle
//   warps 4-7   softmax/epilogue for Q tile A (TMEM lanes 0-127)
//   warps 8-11  softmax/epilogue for Q tile B
// Each item is two GQA-packed Q tiles of 128 rows (G heads x T tokens) that share
// every K/V block in shared memory.  TMEM (512 columns): S_A [0,128) S_B [128,256)
// O_A [256,384) O_B [384,512); P (bf16) is written over its S columns and fed to the
// PV MMA straight from TMEM.
#include <cuda_bf16.h>

#include "kernel_params.h"
#include "ptx.cuh"

namespace ta {

namespace {

template <int D>
struct Cfg {
  static constexpr int kHalves = D / 64;               // 64-column (128 B) swizzle atoms
  static constexpr int kHalfBytes = kTileRows * 128;   // one 64-col region of 128 rows
  static constexpr int kQTileBytes = kTileRows * D * 2;
  static constexpr int kSlotBytes = kBlockKeys * D * 2;  // one K or V block
  static constexpr int kStages = (D == 128) ? 5 : 10;
  static constexpr int kBoxBytes = 64 * 128;          // TMA box: 64 rows x 64 cols bf16
  static constexpr int kBarBytes = 1024;
  static constexpr int kSmem = 1024 /*align slack*/ + 2 * kQTileBytes + kStages * kSlotBytes +
                               kBarBytes;
};

constexpr int kThreads = 384;
constexpr float kRescaleThreshold = 8.0f;  // lazy rescale: exponent headroom in log2 units
constexpr float kLn2 = 0.69314718055994530942f;

struct ItemInfo {
  int kind, kvh, pair;
  int kb0, ke0;   // item key range (band / chunk / causal)
  int r0, r1;     // token rows of the pair, clipped to N
  int s_end, ns;  // sink keys [0, s_end) and their block count (STREAM only)
  int nb;         // total key blocks
};

__device__ __forceinline__ void item_info(const AttnParams &p, const Item &it, ItemInfo &f) {
  f.kind = it.kind;
  f.kvh = it.kv_head;
  f.pair = (int)it.pair;
  f.kb0 = (int)it.key_begin;
  f.ke0 = (int)it.key_end;
  f.r0 = f.pair * p.pair_tokens;
  f.r1 = min(f.r0 + p.pair_tokens, p.n) - 1;
  if (f.kind == kStream) {
    f.s_end = min(p.si, f.r1 + 1);
    f.ns = (f.s_end + kBlockKeys - 1) / kBlockKeys;
  } else {
    f.s_end = 0;
    f.ns = 0;
  }
  f.nb = f.ns + (f.ke0 - f.kb0 + kBlockKeys - 1) / kBlockKeys;
}

// Key block j of an item: first key kb, width n (multiple of 16, <= 128).
__device__ __forceinline__ void block_range(const ItemInfo &f, int j, int &kb, int &n) {
  int e;
  if (j < f.ns) {
    kb = j * kBlockKeys;
    e = f.s_end;
  } else {
    kb = f.kb0 + (j - f.ns) * kBlockKeys;
    e = f.ke0;
  }
  n = min(kBlockKeys, e - kb);
  n = (n + kKeyGranule - 1) & ~(kKeyGranule - 1);
}

__device__ __forceinline__ void ring_pos(uint32_t seq, int stages, uint32_t &slot, uint32_t &ph) {
  slot = seq % (uint32_t)stages;
  ph = (seq / (uint32_t)stages) & 1u;
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1) attn_kernel(const __grid_constant__ AttnParams p) {
  using C = Cfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  uint8_t *sQ = smem;                             // [2][kQTileBytes]
  uint8_t *sKV = smem + 2 * C::kQTileBytes;       // [kStages][kSlotBytes]
  uint64_t *bars = reinterpret_cast<uint64_t *>(sKV + C::kStages * C::kSlotBytes);
  uint64_t *kv_full = bars;
  uint64_t *kv_empty = bars + C::kStages;
  uint64_t *q_full = bars + 2 * C::kStages;
  uint64_t *q_empty = q_full + 1;
  uint64_t *s_full = q_full + 2;   // [2]
  uint64_t *p_ready = q_full + 4;  // [2]
  uint64_t *o_full = q_full + 6;   // [2]
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(q_full + 8);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      ptx::mbar_init(&kv_full[s], 1);
      ptx::mbar_init(&kv_empty[s], 1);
    }
    ptx::mbar_init(q_full, 1);
    ptx::mbar_init(q_empty, 1);
    for (int x = 0; x < 2; ++x) {
      ptx::mbar_init(&s_full[x], 1);
      ptx::mbar_init(&p_ready[x], 128);
      ptx::mbar_init(&o_full[x], 1);
    }
    ptx::fence_mbar_init();
  }
  // Rows >= G*T of a Q tile are never written by TMA: keep them zero.
  for (int i = threadIdx.x; i < 2 * C::kQTileBytes / 16; i += kThreads)
    reinterpret_cast<uint4 *>(sQ)[i] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 2) {
    ptx::tmem_alloc(tmem_slot, 512);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const uint32_t it_beg = p.offsets[blockIdx.x];
  const uint32_t it_end = p.offsets[blockIdx.x + 1];

  if (warp < 4) asm volatile("setmaxnreg.dec.sync.aligned.u32 64;" ::: "memory");

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      ptx::tma_prefetch_desc(&p.tm_q);
      ptx::tma_prefetch_desc(&p.tm_k);
      ptx::tma_prefetch_desc(&p.tm_v);
      uint32_t seq = 0, nitem = 0;
      const uint32_t q_bytes = 2u * C::kHalves * 128u * p.tile_tokens * p.group;
      for (uint32_t ii = it_beg; ii < it_end; ++ii, ++nitem) {
        ItemInfo f;
        item_info(p, p.items[ii], f);
        ptx::mbar_wait(q_empty, (nitem & 1u) ^ 1u);
        ptx::mbar_arrive_expect_tx(q_full, q_bytes);
        for (int x = 0; x < 2; ++x)
          for (int h = 0; h < C::kHalves; ++h)
            ptx::tma_load_3d(sQ + x * C::kQTileBytes + h * C::kHalfBytes, &p.tm_q, q_full, h * 64,
                             f.r0 + x * p.tile_tokens, f.kvh * p.group);
        for (int j = 0; j < f.nb; ++j) {
          int kb, n;
          block_range(f, j, kb, n);
          const int nbox = (n + 63) / 64;
          for (int kv = 0; kv < 2; ++kv, ++seq) {
            uint32_t slot, ph;
            ring_pos(seq, C::kStages, slot, ph);
            ptx::mbar_wait(&kv_empty[slot], ph ^ 1u);
            ptx::mbar_arrive_expect_tx(&kv_full[slot], nbox * C::kHalves * C::kBoxBytes);
            const CUtensorMap *tm = kv ? &p.tm_v : &p.tm_k;
            uint8_t *dst = sKV + slot * C::kSlotBytes;
            for (int h = 0; h < C::kHalves; ++h)
              for (int rb = 0; rb < nbox; ++rb)
                ptx::tma_load_3d(dst + h * C::kHalfBytes + rb * C::kBoxBytes, tm, &kv_full[slot],
                                 h * 64, kb + rb * 64, f.kvh);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      const uint32_t tS[2] = {tmem + 0, tmem + 128};
      const uint32_t tO[2] = {tmem + 256, tmem + 384};
      const uint32_t qbase = ptx::smem_u32(sQ);
      const uint32_t kvbase = ptx::smem_u32(sKV);
      const uint32_t idesc_pv = ptx::idesc_bf16(128, D, 1);
      uint32_t seq = 0, nitem = 0;
      uint32_t pph[2] = {0, 0};
      auto issue_qk = [&](int x, uint32_t kslot, int n) {
        const uint32_t idesc = ptx::idesc_bf16(128, n, 0);
        const uint32_t a0 = qbase + x * C::kQTileBytes;
        const uint32_t b0 = kvbase + kslot * C::kSlotBytes;
#pragma unroll
        for (int s = 0; s < D / 16; ++s) {
          const uint32_t off = (s / 4) * C::kHalfBytes + (s % 4) * 32;
          ptx::mma_ss(tS[x], ptx::sdesc_sw128(a0 + off, 16, 1024),
                      ptx::sdesc_sw128(b0 + off, 16, 1024), idesc, s > 0 ? 1u : 0u);
        }
      };
      auto issue_pv = [&](int x, uint32_t vslot, int n, bool acc) {
        const uint32_t b0 = kvbase + vslot * C::kSlotBytes;
        for (int s = 0; s < n / 16; ++s)
          ptx::mma_ts(tO[x], tS[x] + s * 8, ptx::sdesc_sw128(b0 + s * 2048, C::kHalfBytes, 1024),
                      idesc_pv, (acc || s > 0) ? 1u : 0u);
      };
      for (uint32_t ii = it_beg; ii < it_end; ++ii, ++nitem) {
        ItemInfo f;
        item_info(p, p.items[ii], f);
        ptx::mbar_wait(q_full, nitem & 1u);
        ptx::tc_fence_after();
        const uint32_t seq0 = seq;
        seq += 2u * f.nb;
        uint32_t kslot, kph, vslot, vph;
        int kb, n;
        block_range(f, 0, kb, n);
        ring_pos(seq0, C::kStages, kslot, kph);
        ptx::mbar_wait(&kv_full[kslot], kph);
        ptx::tc_fence_after();
        issue_qk(0, kslot, n);
        ptx::tc_commit(&s_full[0]);
        issue_qk(1, kslot, n);
        ptx::tc_commit(&s_full[1]);
        ptx::tc_commit(&kv_empty[kslot]);
        if (f.nb == 1) ptx::tc_commit(q_empty);
        for (int j = 0; j < f.nb; ++j) {
          const int nj = n;
          ring_pos(seq0 + 2 * j + 1, C::kStages, vslot, vph);
          ptx::mbar_wait(&kv_full[vslot], vph);
          int kb1 = 0, n1 = 0;
          uint32_t kslot1 = 0, kph1 = 0;
          const bool more = (j + 1 < f.nb);
          if (more) {
            block_range(f, j + 1, kb1, n1);
            ring_pos(seq0 + 2 * (j + 1), C::kStages, kslot1, kph1);
          }
          // ---- tile A: PV_A(j), then QK_A(j+1)
          ptx::mbar_wait(&p_ready[0], pph[0]);
          pph[0] ^= 1u;
          ptx::tc_fence_after();
          issue_pv(0, vslot, nj, j > 0);
          if (!more) ptx::tc_commit(&o_full[0]);
          if (more) {
            ptx::mbar_wait(&kv_full[kslot1], kph1);
            ptx::tc_fence_after();
            issue_qk(0, kslot1, n1);
            ptx::tc_commit(&s_full[0]);
          }
          // ---- tile B: PV_B(j), then QK_B(j+1)
          ptx::mbar_wait(&p_ready[1], pph[1]);
          pph[1] ^= 1u;
          ptx::tc_fence_after();
          issue_pv(1, vslot, nj, j > 0);
          if (!more) ptx::tc_commit(&o_full[1]);
          ptx::tc_commit(&kv_empty[vslot]);
          if (more) {
            issue_qk(1, kslot1, n1);
            ptx::tc_commit(&s_full[1]);
            ptx::tc_commit(&kv_empty[kslot1]);
            if (j + 2 == f.nb) ptx::tc_commit(q_empty);
          }
          n = n1;
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ===================== softmax / epilogue =====================
    asm volatile("setmaxnreg.inc.sync.aligned.u32 216;" ::: "memory");
    const int x = (warp - 4) / 4;   // Q tile of this warpgroup
    const int wq = warp % 4;        // TMEM lane quarter
    const int r = wq * 32 + lane;   // packed row = TMEM lane
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    const uint32_t tS = tmem + x * 128 + lane_off;
    const uint32_t tO = tmem + 256 + x * 128 + lane_off;
    const int T = p.tile_tokens;
    const bool row_in_tile = r < p.group * T;
    const int hoff = row_in_tile ? r / T : 0;
    const int toff = row_in_tile ? r % T : 0;
    uint32_t sph = 0, oph = 0;
    for (uint32_t ii = it_beg; ii < it_end; ++ii) {
      ItemInfo f;
      item_info(p, p.items[ii], f);
      const int tok = f.r0 + x * T + toff;     // query row i of this thread
      const bool valid = row_in_tile && tok < p.n;
      // Kept keys of row i inside one key block: [a_lo, a_hi] U [b_lo, b_hi]   (reading R1)
      //   STREAM sink block : j < si, j <= i
      //   STREAM band block : i - sl < j <= i  (band keys are >= si already)
      //   LASTQ             : triangle predicate inside the chunk [kb0, ke0)
      //   DENSE             : j <= i
      // Sink and band blocks may cover the same key numbers (16-key rounding), so each
      // block type keeps only its own section: no pair is counted twice.
      const bool last_row = tok >= p.n - p.last;
      int la_lo, la_hi, lb_lo, lb_hi;  // LASTQ / DENSE intervals
      if (f.kind == kLastQ) {
        la_lo = f.kb0;
        la_hi = last_row ? -1 : min(min(p.si, f.ke0) - 1, tok);
        lb_lo = last_row ? f.kb0 : max(f.kb0, tok - p.sl + 1);
        lb_hi = min(f.ke0 - 1, tok);
      } else {
        la_lo = 0;
        la_hi = -1;
        lb_lo = 0;
        lb_hi = tok;
      }
      float m_run = -INFINITY;  // running max, log2 units of scaled scores
      float l_run = 0.f;        // running sum of 2^(x - m_run)
      for (int j = 0; j < f.nb; ++j) {
        int kb, n;
        block_range(f, j, kb, n);
        const int nch = n / 16;
        ptx::mbar_wait(&s_full[x], sph);
        sph ^= 1u;
        ptx::tc_fence_after();
        float s[128];
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (c < nch) ptx::tmem_ld16f(tS + c * 16, &s[c * 16]);
        ptx::tmem_wait_ld();
        int a_lo = la_lo, a_hi = la_hi, b_lo = lb_lo, b_hi = lb_hi;
        if (f.kind == kStream) {
          if (j < f.ns) {
            a_lo = 0;
            a_hi = min(p.si - 1, tok);
            b_lo = 0;
            b_hi = -1;
          } else {
            a_lo = 0;
            a_hi = -1;
            b_lo = tok - p.sl + 1;
            b_hi = tok;
          }
        }
        const bool full = ((kb >= b_lo) && (kb + n - 1 <= b_hi)) ||
                          ((kb >= a_lo) && (kb + n - 1 <= a_hi));
        const bool warp_full = __all_sync(0xffffffffu, full);
        float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          if (c < nch) {
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const int idx = c * 16 + e;
              float v = s[idx] * p.scale_log2;
              if (!warp_full) {
                const int key = kb + idx;
                const bool kept = (key >= a_lo && key <= a_hi) || (key >= b_lo && key <= b_hi);
                v = kept ? v : -INFINITY;
              }
              s[idx] = v;
              if ((e & 3) == 0) mx0 = fmaxf(mx0, v);
              else if ((e & 3) == 1) mx1 = fmaxf(mx1, v);
              else if ((e & 3) == 2) mx2 = fmaxf(mx2, v);
              else mx3 = fmaxf(mx3, v);
            }
          }
        }
        const float mx = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3));
        const float m_new = fmaxf(m_run, mx);
        const bool need = m_new > m_run + kRescaleThreshold;
        if (__any_sync(0xffffffffu, need)) {
          const float alpha = need ? ptx::ex2(m_run - m_new) : 1.f;
          if (need) m_run = m_new;
          l_run *= alpha;
          if (j > 0) {
            // O_x holds exactly blocks < j: S_x(j) completing implies PV_x(j-1) completed.
#pragma unroll
            for (int c = 0; c < D / 16; ++c) {
              uint32_t o[16];
              ptx::tmem_ld16(tO + c * 16, o, 0);
              ptx::tmem_wait_ld();
#pragma unroll
              for (int e = 0; e < 16; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
              ptx::tmem_st16(tO + c * 16, o);
            }
          }
        }
        const float ref = (m_run == -INFINITY) ? 0.f : m_run;
        float l0 = 0.f, l1 = 0.f, l2 = 0.f, l3 = 0.f;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          if (c < nch) {
            uint32_t pk[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const float a = ptx::ex2(s[c * 16 + 2 * e] - ref);
              const float b = ptx::ex2(s[c * 16 + 2 * e + 1] - ref);
              if (e & 1) {
                l2 += a;
                l3 += b;
              } else {
                l0 += a;
                l1 += b;
              }
              pk[e] = ptx::pack_bf16(a, b);
            }
            ptx::tmem_st8(tS + c * 8, pk);
          }
        }
        l_run += (l0 + l1) + (l2 + l3);
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        ptx::mbar_arrive(&p_ready[x]);
      }
      // ---------------- epilogue
      ptx::mbar_wait(&o_full[x], oph);
      oph ^= 1u;
      ptx::tc_fence_after();
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
      const float lse = l_run > 0.f ? (m_run + __log2f(l_run)) * kLn2 : -INFINITY;
      if (f.kind == kLastQ) {
        const int64_t slot =
            ((int64_t)f.kvh * p.n_last_pairs + (f.pair - p.p_last0)) * p.s_max + f.kb0 / p.chunk_keys;
        const int64_t prow = slot * (2 * kTileRows) + x * kTileRows + r;
        float *dst = p.part_o + prow * D;
#pragma unroll
        for (int c = 0; c < D / 16; ++c) {
          uint32_t o[16];
          ptx::tmem_ld16(tO + c * 16, o, 0);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 16; e += 4) {
            float4 v = make_float4(__uint_as_float(o[e]) * inv, __uint_as_float(o[e + 1]) * inv,
                                   __uint_as_float(o[e + 2]) * inv, __uint_as_float(o[e + 3]) * inv);
            *reinterpret_cast<float4 *>(dst + c * 16 + e) = v;
          }
        }
        p.part_lse[prow] = lse;
      } else {
        const int head = f.kvh * p.group + hoff;
        __nv_bfloat16 *dst = reinterpret_cast<__nv_bfloat16 *>(p.o) +
                             (int64_t)head * p.o_sh + (int64_t)tok * p.o_st;
#pragma unroll
        for (int c = 0; c < D / 16; ++c) {
          uint32_t o[16];
          ptx::tmem_ld16(tO + c * 16, o, 0);
          ptx::tmem_wait_ld();
          uint32_t pk[8];
#pragma unroll
          for (int e = 0; e < 8; ++e)
            pk[e] = ptx::pack_bf16(__uint_as_float(o[2 * e]) * inv, __uint_as_float(o[2 * e + 1]) * inv);
          if (valid) {
            uint4 *d4 = reinterpret_cast<uint4 *>(dst + c * 16);
            d4[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            d4[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
          }
        }
        if (valid && p.lse) p.lse[(int64_t)head * p.n + tok] = lse;
      }
      ptx::tc_fence_before();
    }
  }
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

// One warp per packed row of a last pair: O = sum_c e^{LSE_c - M} O_c / sum_c e^{LSE_c - M}
// over the pair's split-K chunks (merge_output; reading R8/R18).
template <int D>
__global__ void __launch_bounds__(256) merge_kernel(const __grid_constant__ AttnParams p) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t gw = (int64_t)blockIdx.x * 8 + warp;  // (kvh, last pair, row) linear
  const int rows = 2 * kTileRows;
  const int64_t per_kvh = (int64_t)p.n_last_pairs * rows;
  const int kvh = (int)(gw / per_kvh);
  const int rem = (int)(gw % per_kvh);
  const int lp = rem / rows, rr = rem % rows;
  if (kvh >= p.hq / p.group) return;
  const int x = rr / kTileRows, r = rr % kTileRows;
  const int T = p.tile_tokens;
  if (r >= p.group * T) return;
  const int pair = p.p_last0 + lp;
  const int tok = pair * p.pair_tokens + x * T + r % T;
  if (tok >= p.n) return;
  const int head = kvh * p.group + r / T;
  const int r1 = min((pair + 1) * p.pair_tokens, p.n) - 1;
  const int nch = (r1 + 1 + p.chunk_keys - 1) / p.chunk_keys;
  const int64_t slot0 = ((int64_t)kvh * p.n_last_pairs + lp) * p.s_max;
  float mx = -INFINITY;
  for (int c = lane; c < nch; c += 32) mx = fmaxf(mx, p.part_lse[(slot0 + c) * rows + rr]);
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  constexpr int E = D / 32;
  float acc[E];
#pragma unroll
  for (int e = 0; e < E; ++e) acc[e] = 0.f;
  float wsum = 0.f;
  for (int c = 0; c < nch; ++c) {
    const float lc = p.part_lse[(slot0 + c) * rows + rr];
    if (lc == -INFINITY) continue;  // empty chunk: weight 0, never exp(-inf - -inf)
    const float w = __expf(lc - mx);
    wsum += w;
    const float *src = p.part_o + ((slot0 + c) * rows + rr) * D;
#pragma unroll
    for (int e = 0; e < E; ++e) acc[e] += w * src[lane + 32 * e];
  }
  const float inv = wsum > 0.f ? 1.f / wsum : 0.f;
  __nv_bfloat16 *dst = reinterpret_cast<__nv_bfloat16 *>(p.o) + (int64_t)head * p.o_sh +
                       (int64_t)tok * p.o_st;
#pragma unroll
  for (int e = 0; e < E; ++e) dst[lane + 32 * e] = __float2bfloat16_rn(acc[e] * inv);
  if (lane == 0 && p.lse) p.lse[(int64_t)head * p.n + tok] = wsum > 0.f ? mx + __logf(wsum) : -INFINITY;
}

}  // namespace

size_t attention_smem_bytes(int head_dim) {
  return head_dim == 128 ? Cfg<128>::kSmem : Cfg<64>::kSmem;
}

template <int D>
static cudaError_t launch_attention_t(const AttnParams &p, int num_ctas, cudaStream_t s) {
  static bool attr_set = false;  // per-process; cudaFuncSetAttribute is cheap and idempotent
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(attn_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg<D>::kSmem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  attn_kernel<D><<<num_ctas, kThreads, Cfg<D>::kSmem, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_attention(const AttnParams &p, int head_dim, int num_ctas, cudaStream_t s) {
  return head_dim == 128 ? launch_attention_t<128>(p, num_ctas, s)
                         : launch_attention_t<64>(p, num_ctas, s);
}

cudaError_t launch_merge(const AttnParams &p, int head_dim, int hkv, cudaStream_t s) {
  const int64_t rows = (int64_t)hkv * p.n_last_pairs * 2 * kTileRows;
  const unsigned blocks = (unsigned)((rows + 7) / 8);
  if (blocks == 0) return cudaSuccess;
  if (head_dim == 128)
    merge_kernel<128><<<blocks, 256, 0, s>>>(p);
  else
    merge_kernel<64><<<blocks, 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace ta
