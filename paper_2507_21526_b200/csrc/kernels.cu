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
// CTA layout (512 threads, 1 CTA per SM):
//   warps 0-3   epilogue warpgroup (O normalisation + TMA stores, both tiles in turn)
//   warps 4-7   softmax for Q tile A (TMEM lanes 0-127)
//   warps 8-11  softmax for Q tile B
//   warp 12     MMA issuer  (whole warp, one elected lane issues)
//   warp 13     TMA producer
//   warp 14     TMEM allocator, warp 15 idle
// Each item is two GQA-packed Q tiles of 128 rows (G heads x T tokens) that share
// every K/V block in shared memory.  TMEM (512 columns): S_A [0,128) S_B [128,256)
// O_A [256,384) O_B [384,512); P (bf16) is written over its S columns and fed to the
// PV MMA straight from TMEM.
//
// Sink fusion: when a STREAM item's sink span is <= 16 keys (si = 8 in the paper,
// P:L295) the sink K/V rows are loaded with the Q tiles into a 16-row side buffer and
// occupy S columns [0,16) of the first key block, whose remaining 112 columns hold the
// start of the sliding-window band.
#include <cuda_bf16.h>

#include <atomic>
#include <cstdlib>
#include <type_traits>

#include "kernel_params.h"
#include "ptx.cuh"

namespace ta {

namespace {

#ifdef TA_TRACE
// Debug timeline (builds with -DTA_TRACE only): clock64 stamps of one CTA's pipeline events.
#define TRACE_AT(base, cnt, code, arg)                                                       \
  do {                                                                                       \
    if (p.trace && blockIdx.x == (unsigned)p.trace_cta && cnt < 65535)                       \
      p.trace[(base) + (cnt)++] = ((uint64_t)(code) << 56) | ((uint64_t)((arg) & 0xff) << 48) | \
                                  ((uint64_t)clock64() & 0xffffffffffffull);                  \
  } while (0)
#define TRACE_PR(code, arg) do { if (leader) TRACE_AT(0, trc, code, arg); } while (0)
#define TRACE_MM(code, arg) do { if (leader) TRACE_AT(65536, trc, code, arg); } while (0)
#define TRACE_SM(code, arg) do { if (lane == 0 && wq == 0 && hc == 0) TRACE_AT(131072 + 65536 * x, trc, code, arg); } while (0)
// tile A warps 1-3 (drift across the four warps of a tile): roles 5-7
#define TRACE_SMW(code, arg) do { if (lane == 0 && x == 0 && wq > 0 && hc == 0) TRACE_AT(65536 * (4 + wq), trc, code, arg); } while (0)
#define TRACE_EP(code, arg) do { if (lane == 0 && eq == 0 && x0 == 0) TRACE_AT(262144, trc, code, arg); } while (0)
#else
#define TRACE_PR(code, arg) do {} while (0)
#define TRACE_MM(code, arg) do {} while (0)
#define TRACE_SM(code, arg) do {} while (0)
#define TRACE_SMW(code, arg) do {} while (0)
#define TRACE_EP(code, arg) do {} while (0)
#endif

template <int D>
struct Cfg {
  static constexpr int kHalves = D / 64;                 // 64-column (128 B) swizzle atoms
  static constexpr int kHalfBytes = kTileRows * 128;     // one 64-col region of 128 rows
  static constexpr int kQTileBytes = kTileRows * D * 2;
  // A K or V slot: per 64-column half, 128 key rows (a fused first block puts 16 sink rows
  // in front of 112 band rows).
  static constexpr int kSlotRows = kBlockKeys;
  static constexpr int kSlotHalfBytes = kSlotRows * 128;
  static constexpr int kSlotBytes = kHalves * kSlotHalfBytes;
  static constexpr int kStages = (D == 128) ? 4 : 8;
  static constexpr int kBarBytes = 1024;
  static constexpr int kRedBytes = 2 * 2 * 2 * kTileRows * 4 * 2 + 2 * 2 * kTileRows * 4;
  static constexpr int kStageBytes = 128 * 128;  // epilogue: one 64-column half of an O tile (bf16, SW128)
  static constexpr int kSmem = 1024 /*align slack*/ + 2 * kQTileBytes + kStages * kSlotBytes +
                               kBarBytes + kRedBytes + kStageBytes;
};

// Warp roles.  Softmax: kHPR threads per query row (128 / kHPR columns each), 4 kHPR
// warps per Q tile (tile A first); then the epilogue warpgroup (TMEM lane quarters 0-3),
// then the MMA issuer, TMA producer and TMEM allocator.  Higher warp ids win the
// highest-warp-id-first issue arbitration, so the issuers and the epilogue are never
// starved by the softmax warps.
#ifndef TA_HPR
#define TA_HPR 1
#endif
constexpr int kHPR = TA_HPR;
constexpr int kSoftmaxWarps = 8 * kHPR;
#ifndef TA_EPI_WARPS  // epilogue warps: 4 per Q tile (TA_EPI_WARPS = 8) or 4 serving both tiles in turn
#define TA_EPI_WARPS 4
#endif
constexpr int kEpiWarps = TA_EPI_WARPS;
// TA_EPI_LOW: the epilogue warpgroup takes warps 0-3 and the softmax warps 4-11, so the
// softmax (the critical path) wins issue arbitration over the epilogue on every SMSP.
#ifndef TA_EPI_LOW
#define TA_EPI_LOW 1
#endif
constexpr bool kEpiLow = TA_EPI_LOW != 0 && kHPR == 1 && kEpiWarps == 4;
constexpr int kSmWarp0 = kEpiLow ? kEpiWarps : 0;
constexpr int kEpiWarp0 = kEpiLow ? 0 : kSoftmaxWarps;
// Issuer warps: the four warps after the softmax and epilogue warps.  TA_MMA_SLOT picks the
// MMA issuer's SM sub-partition (warp % 4): 0 shares SMSP 0 with the epilogue's store-issuing
// warp; the TMA producer and TMEM allocator take the next slots.
#ifndef TA_MMA_SLOT
#define TA_MMA_SLOT 0
#endif
constexpr int kIssuer0 = kSoftmaxWarps + kEpiWarps;
constexpr int kMmaWarp = kIssuer0 + TA_MMA_SLOT;
constexpr int kTmaWarp = kIssuer0 + (TA_MMA_SLOT + 1) % 4;
constexpr int kAllocWarp = kIssuer0 + (TA_MMA_SLOT + 2) % 4;
constexpr int kThreads = 32 * (kSoftmaxWarps + kEpiWarps + 4);
// 1 (default): no item_empty hand-back.  Slot reuse is safe by the pipeline's own back-
// pressure: the producer publishes item k+1 only after issuing item k's K/V loads (4-slot
// ring = 2 blocks) and item k's Q (waits for item k-1's last QK^T), so it leads the MMA warp
// by <= 2 items; the MMA leads the softmax by <= 1 (QK^T(j+1) waits for P(j)) and the
// softmax leads the epilogue by <= 2 (it publishes item k after o_free of item k-1): <= 5
// items in flight against 16 ring entries.  (0: per-slot empty barriers; +0.3 % cycles.)
#ifndef TA_RING_NOEMPTY
#define TA_RING_NOEMPTY 1
#endif
constexpr int kItemRing = TA_RING_NOEMPTY ? 16 : 8;  // published entries (roles lag the producer by <= ~3)
constexpr int kItemConsumers = 1 + kSoftmaxWarps + kEpiWarps;  // MMA warp + softmax + epilogue warps
constexpr int kNCol = 128 / kHPR;  // S columns per softmax thread
// setmaxnreg split of the register file (launch: 65536 / kThreads, rounded down to 8)
#ifndef TA_REG_SOFTMAX
#define TA_REG_SOFTMAX 176
#endif
constexpr int kRegSoftmax = kEpiWarps == 4 ? (kHPR == 1 ? TA_REG_SOFTMAX : 96) : (kHPR == 1 ? 176 : 88);
#ifndef TA_REG_EPI  // epilogue warpgroup; the issuer warpgroup gets the rest (2 S + E + O = 512)
#define TA_REG_EPI ((2048 - 8 * TA_REG_SOFTMAX) / 8)
#endif
constexpr int kRegEpi = kEpiWarps == 4 ? (kHPR == 1 ? TA_REG_EPI : 48) : 40;
constexpr int kRegOther = kEpiWarps == 4 ? (kHPR == 1 ? 512 - 2 * TA_REG_SOFTMAX - TA_REG_EPI : 48)
                                         : (kHPR == 1 ? 48 : 40);
static_assert(kRegOther >= 24 && kRegOther % 8 == 0 && kRegEpi % 8 == 0, "setmaxnreg split");
#ifndef TA_WARP_ARRIVE
#define TA_WARP_ARRIVE 0
#endif
constexpr int kArrivePerTile = TA_WARP_ARRIVE ? 4 : kTileRows;  // softmax arrivals per tile
constexpr float kRescaleThreshold = 8.0f;  // lazy rescale: exponent headroom in log2 units
constexpr float kLn2 = 0.69314718055994530942f;
constexpr int kEmpty = 1 << 30;            // canonical empty column interval [kEmpty, kEmpty]
// Bit k set: column pair k (of the 8 pairs in every 16 columns) uses the FMA-pipe exp2
// instead of MUFU.EX2.  Default 0: every exponential on MUFU -- with the exp phase bound by
// the FMA pipe (FFMA2 scale, FADD2 row sum, F2FP) the offload measured slower (cycles per
// item: 0x25 +2.4 %, 0x11 +2.2 %, 0x01 +0.5 % vs 0x00; scripts/variant_cycles.py).
// Row sum l (the softmax denominator): 4 (default) = the bf16-rounded P that the PV MMA
// consumes, added with mixed-precision FHADD.BF16 (exact normalisation: V = 1 gives O = 1,
// and a row dominated by one key carries no P-rounding mismatch between O and l; +3.1 %
// cycles at C3 vs the fp32 sum).  0 = fp32 p (FADD2); 1 / 2 = unpack the bf16 pair
// (IMAD.SHL + LOP3 / PRMT + LOP3) + FADD2 (+9 % / +10 %); 3 = truncate P on the ALU pipe
// (+7.6 %).  Measured with scripts/variant_ctaclk.py.
#ifndef TA_SUM_ROUNDED
#define TA_SUM_ROUNDED 4
#endif
#ifndef TA_FHADD_ACC  // independent FHADD accumulators per row (2: -0.5 % cycles vs 4)
#define TA_FHADD_ACC 2
#endif
#ifndef TA_SM_WAIT
#define TA_SM_WAIT 0
#endif
#ifndef TA_TILE_TRIM
#define TA_TILE_TRIM 0
#endif
#ifndef TA_POLY_DEG
#define TA_POLY_DEG 3
#endif
#ifndef TA_POLY_MASK
#define TA_POLY_MASK 0x01
#endif
constexpr int kPolyPairs = TA_POLY_MASK;
// MMA issuer barrier waits: suspending try_wait (default) or a test_wait spin
#if defined(TA_MMA_SPIN) && !defined(TA_WATCHDOG)
#define MMA_WAIT(bar, ph) ptx::mbar_wait_spin(bar, ph)
#else
#define MMA_WAIT(bar, ph) ptx::mbar_wait(bar, ph)
#endif
#ifndef TA_TMEM_WIDE
#define TA_TMEM_WIDE 1
#endif
#ifndef TA_EXP_ORDER
#define TA_EXP_ORDER 1
#endif
#ifndef TA_MMA_REMAT
#define TA_MMA_REMAT 1
#endif
#ifndef TA_EXTRA_WAITS
#define TA_EXTRA_WAITS 0
#endif
#ifndef TA_PV_SPLIT  // PV in two halves, the first on p_ready (keys 0..63) mid-softmax
#define TA_PV_SPLIT 1
#endif
#ifndef TA_EARLY_K
#define TA_EARLY_K 0
#endif
#ifndef TA_SPLIT  // 16-column chunks of P handed to the MMA first (p_ready); even, <= 8
#define TA_SPLIT 4
#endif
constexpr int kSplit = TA_SPLIT;
static_assert(kSplit % 2 == 0 && kSplit >= 2 && kSplit <= 8, "P hand-off split");
// Timing-only experiments (wrong results; never in a shipped build): skip the epilogue's
// work (NOEPI) or load Q only for a CTA's first item (QONCE).
#ifndef TA_EXP_NOEPI
#define TA_EXP_NOEPI 0
#endif
#ifndef TA_EXP_QONCE
#define TA_EXP_QONCE 0
#endif
#ifndef TA_COLD_START  // first item: Q and K0 first, the rest of the ring after Q has landed
#define TA_COLD_START 1
#endif
#ifndef TA_EXP_QKEARLY  // timing probe (wrong results): QK^T(next) issued before PV (chain length)
#define TA_EXP_QKEARLY 0
#endif
#ifndef TA_EXP_NOMASK  // timing only: no kept-column masking (wrong results)
#define TA_EXP_NOMASK 0
#endif
#ifndef TA_SKIP_RAGGED  // exponentials only over the block's computed 16-column chunks
#define TA_SKIP_RAGGED 0
#endif
#ifndef TA_MASK_VOTE
#define TA_MASK_VOTE 0
#endif
#ifndef TA_SHORT_BODY  // blocks of <= 80 S columns run a 5-chunk softmax body (see below)
#define TA_SHORT_BODY 1
#endif
#ifndef TA_SHORT_STREAM_ONLY  // the short body only for STREAM items (not DENSE / LASTQ blocks)
#define TA_SHORT_STREAM_ONLY 0
#endif
#ifndef TA_SHORT4  // a third, 4-chunk body for blocks of <= 64 columns (Qwen: P = 36)
#define TA_SHORT4 0
#endif
#ifndef TA_EPI_FMUL2
#define TA_EPI_FMUL2 0
#endif
#ifndef TA_PINGPONG
#define TA_PINGPONG 0
#endif
constexpr bool kPingPong = TA_PINGPONG != 0;

// Causal-profiling debug switches: spin N cycles at a point of one role per key block.
#ifndef TA_DELAY_MMA
#define TA_DELAY_MMA 0
#endif
#ifndef TA_DELAY_SM
#define TA_DELAY_SM 0
#endif
#ifndef TA_DELAY_TMA
#define TA_DELAY_TMA 0
#endif
// Wait accounting (TA_WAITSTAT builds, with TA_CTA_CLOCK): each role sums the SM cycles it
// spends in each barrier wait (and the MMA issuer in its issue loops); written at the end
// to trace[4096 + 128 cta + 16 role + k]
// (roles: 0 TMA producer, 1 MMA issuer, 2/3 softmax tile A/B (warp quarter 0, lane 0),
// 4 epilogue (warp 0, lane 0)); scripts/waitstat.py prints them.
#ifdef TA_WAITSTAT
#define WS_DECL long long ws_acc[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}
#define WS(k, ...)                          \
  do {                                      \
    const long long ws_t0_ = clock64();     \
    __VA_ARGS__;                            \
    ws_acc[k] += clock64() - ws_t0_;        \
  } while (0)
#define WS_DUMP(role, cond)                                                          \
  do {                                                                              \
    if (cond)                                                                       \
      for (int k_ = 0; k_ < 16; ++k_) p.trace[4096 + 128 * blockIdx.x + 16 * (role) + k_] = ws_acc[k_]; \
  } while (0)
#else
#define WS_DECL
#define WS(k, ...) \
  do {             \
    __VA_ARGS__;   \
  } while (0)
#define WS_DUMP(role, cond) \
  do {                      \
  } while (0)
#endif

__device__ __forceinline__ void spin_cycles(int n) {
  if (n > 0) {
    const long long t0 = clock64();
    while (clock64() - t0 < n) {
    }
  }
}

struct ItemInfo {
  int kind, kvh, pair;
  int kb0, ke0;   // item key range (band / chunk / causal)
  int r0, r1;     // token rows of the pair, clipped to N
  int fused;      // STREAM: sink (<= 16 keys) folded into block 0
  int chunk;      // LASTQ: piece index within the pair's span (split-K slot)
  int s_end, ns;  // STREAM unfused: sink keys [0, s_end) in ns blocks of their own
  int nb;         // total key blocks
};

struct Blk {
  int kb;     // first key of the K/V slot rows
  int nk;     // keys loaded into the slot (<= 128)
  int sink;   // sink columns in front (0 or 16)
  int ncols;  // total S columns (multiple of 16, <= 128)
  int sinkblk;  // unfused sink block
};

__device__ __forceinline__ int ceil_div(int a, int b) { return (a + b - 1) / b; }
__device__ __forceinline__ int round16(int a) { return (a + 15) & ~15; }

__device__ __forceinline__ void item_info(const AttnParams &p, const Item &it, ItemInfo &f) {
  f.kind = it.kind;
  f.kvh = it.kv_head;
  f.pair = (int)it.pair;
  f.kb0 = (int)it.key_begin;
  f.ke0 = (int)it.key_end;
  f.chunk = it.pad;
  f.r0 = f.pair * p.pair_tokens;
  f.r1 = min(f.r0 + p.pair_tokens, p.n) - 1;
  f.fused = 0;
  f.s_end = 0;
  f.ns = 0;
  const int len = f.ke0 - f.kb0;
  if (f.kind == kStream) {
    f.s_end = min(p.si, f.r1 + 1);
    if (f.s_end > 0 && f.s_end <= kSinkRows) {
      f.fused = 1;
      const int first = kBlockKeys - kSinkRows;
      f.nb = 1 + (len > first ? ceil_div(len - first, kBlockKeys) : 0);
      return;
    }
    f.ns = ceil_div(f.s_end, kBlockKeys);
  }
  f.nb = f.ns + ceil_div(len, kBlockKeys);
}

__device__ __forceinline__ Blk block_info(const ItemInfo &f, int j) {
  Blk b;
  b.sink = 0;
  b.sinkblk = 0;
  if (f.fused) {
    if (j == 0) {
      b.kb = f.kb0;
      b.nk = min(kBlockKeys - kSinkRows, f.ke0 - f.kb0);
      b.sink = kSinkRows;
    } else {
      b.kb = f.kb0 + (kBlockKeys - kSinkRows) + (j - 1) * kBlockKeys;
      b.nk = min(kBlockKeys, f.ke0 - b.kb);
    }
  } else if (j < f.ns) {
    b.kb = j * kBlockKeys;
    b.nk = min(kBlockKeys, f.s_end - b.kb);
    b.sinkblk = 1;
  } else {
    b.kb = f.kb0 + (j - f.ns) * kBlockKeys;
    b.nk = min(kBlockKeys, f.ke0 - b.kb);
  }
  b.ncols = b.sink + round16(b.nk);
  return b;
}

// S columns Q tile x needs in block b: every kept key satisfies j <= i, and the largest
// token of tile x is r0 + (x+1) T - 1, so the tail of a block beyond it is masked for the
// whole tile and its QK^T / softmax / PV are skipped (>= 16 columns, <= b.ncols).
__device__ __forceinline__ int tile_ncols(const ItemInfo &f, const Blk &b, int x, int T) {
#if TA_TILE_TRIM
  const int rmax = f.r0 + (x + 1) * T - 1;
  const int nk = max(1, min(b.nk, rmax - b.kb + 1));
  return b.sink + round16(nk);
#else
  return b.ncols;
#endif
}

__device__ __forceinline__ void ring_pos(uint32_t seq, int stages, uint32_t &slot, uint32_t &ph) {
  slot = seq % (uint32_t)stages;
  ph = (seq / (uint32_t)stages) & 1u;
}

// ---- packed fp32x2 helpers (FFMA2 / FADD2 on sm_100a)
__device__ __forceinline__ uint64_t f2pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2unpack(uint64_t v, float &lo, float &hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ float max3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// (a << 23) + b with shift+add on the integer ALU pipe (keeps the FMA pipe for FFMA2).
__device__ __forceinline__ int lea23(int a, int b) {
  int r;
  asm("{\n\t.reg .b32 t;\n\tshl.b32 t, %1, 23;\n\tadd.s32 %0, t, %2;\n\t}" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

// 2^x for a pair on the FMA pipe (offloads the MUFU unit): x = j + f, j = rint(x),
// f in [-1/2, 1/2], 2^f ~ 1 + c1 f + c2 f^2 + c3 f^3 (max rel. err 1.0e-4, far below the
// bf16 rounding of P).  x is clamped to >= -127 so that x = -inf (a masked score) gives
// exactly +0: p(0) = 1 and 1 * 2^-127 encodes as 0x00000000.
__device__ __forceinline__ void exp2_poly2(float x0, float x1, float &y0, float &y1) {
  constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23: rint via fp add
  x0 = fmaxf(x0, -127.f);
  x1 = fmaxf(x1, -127.f);
  const uint64_t x = f2pack(x0, x1);
  const uint64_t t = fadd2(x, f2pack(kMagic, kMagic));
  const uint64_t r = fadd2(t, f2pack(-kMagic, -kMagic));
  uint64_t f = ffma2(r, f2pack(-1.f, -1.f), x);    // x - rint(x), exact
  uint64_t pp;
  if (TA_POLY_DEG == 3) {
    pp = ffma2(f, f2pack(0.055008280f, 0.055008280f), f2pack(0.24220959f, 0.24220959f));
    pp = ffma2(pp, f, f2pack(0.69328285f, 0.69328285f));
  } else {  // degree 2: max rel. err 2.0e-3 (about the bf16 rounding of P)
    pp = ffma2(f, f2pack(0.23985499f, 0.23985499f), f2pack(0.70292904f, 0.70292904f));
  }
  pp = ffma2(pp, f, f2pack(1.0f, 1.0f));
  float p0, p1, t0, t1;
  f2unpack(pp, p0, p1);
  f2unpack(t, t0, t1);
  y0 = __int_as_float(lea23(__float_as_int(t0), __float_as_int(p0)));
  y1 = __int_as_float(lea23(__float_as_int(t1), __float_as_int(p1)));
}

__device__ __forceinline__ uint64_t u2pack(uint32_t lo, uint32_t hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
  return r;
}

#if TA_SUM_ROUNDED == 2 || TA_SUM_ROUNDED == 3
// bf16 bit helpers pinned to the integer ALU pipe (the compiler would otherwise emit
// IMAD.SHL on the FMA pipe, which the exponential phase already saturates).
__device__ __forceinline__ uint32_t hi16(uint32_t a) {  // a & 0xffff0000 (LOP3)
  uint32_t r;
  asm("and.b32 %0, %1, 0xffff0000;" : "=r"(r) : "r"(a));
  return r;
}
__device__ __forceinline__ uint32_t lo16_up(uint32_t a) {  // a << 16 (PRMT)
  uint32_t r;
  asm("prmt.b32 %0, %1, 0, 0x1044;" : "=r"(r) : "r"(a));
  return r;
}
__device__ __forceinline__ uint32_t prmt_hi(uint32_t lo, uint32_t hi) {  // {hi.hi16, lo.hi16}
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(lo), "r"(hi));
  return r;
}
#endif
__device__ __forceinline__ void sum_bf16_lo(float &acc, uint32_t pk) {
  asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %1;\n\tadd.rn.f32.bf16 %0, l, %0;\n\t}" : "+f"(acc) : "r"(pk));
}
__device__ __forceinline__ void sum_bf16_hi(float &acc, uint32_t pk) {
  asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %1;\n\tadd.rn.f32.bf16 %0, h, %0;\n\t}" : "+f"(acc) : "r"(pk));
}

// Bits [lo, hi] of a 32-bit word (empty if hi < lo or outside [0, 31]).
__device__ __forceinline__ uint32_t iv_bits(int lo, int hi) {
  lo = max(lo, 0);
  hi = min(hi, 31);
  if (hi < lo) return 0u;
  const uint32_t upto_hi = (hi == 31) ? 0xffffffffu : ((2u << hi) - 1u);
  return upto_hi & ~((1u << lo) - 1u);
}


__device__ __forceinline__ void sts_f32(uint32_t a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts_v4(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w)
               : "memory");
}


// 256-bit global store (STG.E.256 on sm_100a); p must be 32-byte aligned.
__device__ __forceinline__ void st_global_v8(void *p, const uint32_t *v) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}

// Normalise a column interval; empty -> [kEmpty, kEmpty].
__device__ __forceinline__ void norm_iv(int &lo, int &hi) {
  if (lo > hi) {
    lo = kEmpty;
    hi = kEmpty;
  }
}

// Tail ticket that carried another launch's epoch (it reached the queue word before CTA 0's
// reset): wait and retry until the reset has landed.  Out of line: never taken in practice.
__device__ __noinline__ unsigned long long stale_ticket_retry(uint32_t *queue, uint32_t epoch) {
  unsigned long long v;
  do {
    __nanosleep(256);
    v = atomicAdd(reinterpret_cast<unsigned long long *>(queue), 1ull);
  } while ((v >> 32) != epoch);
  return v;
}

// 16-byte store to a multicast (NVLS) address: one egress, every bound GPU receives it.
__device__ __forceinline__ void mc_st16(void *p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("multimem.st.global.v4.bf16x2 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}
__device__ __forceinline__ void mc_st4(void *p, uint32_t a) {
  asm volatile("multimem.st.global.bf16x2 [%0], %1;" ::"l"(p), "r"(a) : "memory");
}

// Output modes.  The f2 entry points get their own instantiations, so the single-output
// epilogue -- on the kernel's critical path -- carries no destination code (a destination
// loop compiled into it measured +2.5 % cycles).
constexpr int kOutSingle = 0;     // TMA store to p.o
constexpr int kOutExtra = 1;      // + TMA stores to up to 7 extra destinations (unicast)
constexpr int kOutMulticast = 2;  // + 16-byte multimem stores to the multicast view p.mc_o
template <int D, int kMode>
__global__ void __launch_bounds__(kThreads, 1) attn_kernel(const __grid_constant__ AttnParams p) {
  using C = Cfg<D>;
#if defined(TA_CTA_CLOCK) && defined(TA_GT)
  unsigned long long cta_g0;  // globaltimer at kernel entry (before the prologue)
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(cta_g0));
#endif
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  uint8_t *sQ = smem;                                   // [2][kQTileBytes]
  uint8_t *sKV = smem + 2 * C::kQTileBytes;              // [kStages][kSlotBytes]
  uint64_t *bars = reinterpret_cast<uint64_t *>(sKV + C::kStages * C::kSlotBytes);
  uint64_t *kv_full = bars;
  uint64_t *kv_empty = bars + C::kStages;
  uint64_t *q_full = bars + 2 * C::kStages;
  uint64_t *q_empty = q_full + 1;
  uint64_t *s_full = q_full + 2;   // [2]
  uint64_t *p_ready = q_full + 4;  // [2]
  uint64_t *o_full = q_full + 6;   // [2]
  uint64_t *exp_turn = q_full + 8;  // [2] softmax ping-pong: tile x may run its exp phase
  uint64_t *l_ready = q_full + 10;  // [2] softmax -> epilogue: row sums / max of an item written
  uint64_t *o_free = q_full + 12;   // [2] epilogue -> MMA: O_x drained from TMEM
  uint64_t *p_hi = q_full + 14;     // [2] P of keys 64..127 written (p_ready: keys 0..63)
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(q_full + 16);
  // Dynamic work queue: the TMA producer fetches item indices (global atomic counter, in the
  // schedule's fetch order) and publishes them in a ring the other roles read in sequence.
  uint64_t *item_full = q_full + 18;          // [kItemRing], 1 arrival (producer)
  uint64_t *item_empty = item_full + kItemRing;  // [kItemRing], kItemConsumers arrivals
  volatile int32_t *item_ring = reinterpret_cast<volatile int32_t *>(item_empty + kItemRing);
  // cross-warp row reductions of the two column halves of a row:
  // red_max[tile][block parity][half][row]; red_l[item parity][tile][half][row];
  // red_m[item parity][tile][row]
  float *red_max = reinterpret_cast<float *>(reinterpret_cast<uint8_t *>(bars) + C::kBarBytes);
  float *red_l = red_max + 2 * 2 * 2 * kTileRows;
  float *red_m = red_l + 2 * 2 * 2 * kTileRows;
  uint8_t *stage = reinterpret_cast<uint8_t *>(red_m + 2 * 2 * kTileRows);  // 1024-aligned, 16 KB

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
      ptx::mbar_init(&p_ready[x], kArrivePerTile);  // first 64 keys of P written
      ptx::mbar_init(&p_hi[x], kArrivePerTile);     // last 64 keys of P written
      ptx::mbar_init(&o_full[x], 1);
      ptx::mbar_init(&exp_turn[x], 4 * kHPR);  // one arrival per softmax warp of the other tile
      ptx::mbar_init(&l_ready[x], kHPR * kArrivePerTile);
      ptx::mbar_init(&o_free[x], 4);     // one arrival per epilogue warp
    }
    for (int r = 0; r < kItemRing; ++r) {
      ptx::mbar_init(&item_full[r], 1);
      ptx::mbar_init(&item_empty[r], kItemConsumers);
    }
    ptx::fence_mbar_init();
  }
  // Rows >= G*T of a Q tile are never written by TMA: keep them zero (only when G*T < 128,
  // e.g. Qwen's G = 7; a full tile is overwritten by every Q load).
  if (p.group * p.tile_tokens < kTileRows)
    for (int i = threadIdx.x; i < 2 * C::kQTileBytes / 16; i += kThreads)
      reinterpret_cast<uint4 *>(sQ)[i] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == kAllocWarp) {
    ptx::tmem_alloc(tmem_slot, 512);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  // TMEM base: every role re-reads it from shared memory where it starts (a kernel-wide live
  // value ends up spilled and reloaded on the MMA issue path)
  auto tmem_base = [&]() -> uint32_t {
    uint32_t t;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(t) : "r"(ptx::smem_u32(tmem_slot)) : "memory");
    return t;
  };

#ifdef TA_CTA_CLOCK
  const long long cta_t0 = clock64();
#endif
  // Consumer side of the work queue: the item index of this CTA's k-th item (-1: no more).
  auto take_item = [&](uint32_t k) -> int {
    const uint32_t slot = k % kItemRing;
    ptx::mbar_wait(&item_full[slot], (k / kItemRing) & 1u);
    const int idx = item_ring[slot];
    if (!TA_RING_NOEMPTY) {
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&item_empty[slot]);
    }
    return idx;
  };

  // Register split: softmax warpgroups kRegSoftmax, epilogue kRegEpi, issuers kRegOther.
  if (warp >= kIssuer0) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegOther) : "memory");
  else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + kEpiWarps)
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegEpi) : "memory");

  if (warp == kTmaWarp) {
    // ===================== TMA producer (whole warp, one elected lane issues) ==========
    const bool leader = ptx::elect_one();
    WS_DECL;
    {
#ifdef TA_TRACE
      uint32_t trc = 0;
#endif
      if (leader) {
        ptx::tma_prefetch_desc(&p.tm_q);
        ptx::tma_prefetch_desc(&p.tm_k);
        ptx::tma_prefetch_desc(&p.tm_v);
      }
      uint32_t seq = 0, nitem = 0;
      const uint32_t q_bytes = 2u * C::kHalves * 128u * p.tile_tokens * p.group;
      auto load_q = [&](const ItemInfo &f, uint32_t nitem) {
        WS(0, ptx::mbar_wait_lazy(q_empty, (nitem & 1u) ^ 1u));
        if (leader) {
          ptx::mbar_arrive_expect_tx(q_full, q_bytes);
          for (int x = 0; x < 2; ++x)
            for (int h = 0; h < C::kHalves; ++h)
              ptx::tma_load_3d(sQ + x * C::kQTileBytes + h * C::kHalfBytes, &p.tm_q, q_full, h * 64,
                               f.r0 + x * p.tile_tokens, f.kvh * p.group);
          TRACE_PR(1, nitem);
        }
      };
      // K (kv = 0) and / or V (kv = 1) of block j, each into the next ring slot
      auto load_kv = [&](const ItemInfo &f, int j, int kv0 = 0, int kv1 = 2) {
        spin_cycles(TA_DELAY_TMA);
        const Blk b = block_info(f, j);
        for (int kv = kv0; kv < kv1; ++kv, ++seq) {
          uint32_t slot, ph;
          ring_pos(seq, C::kStages, slot, ph);
          WS(1, ptx::mbar_wait_lazy(&kv_empty[slot], ph ^ 1u));
          if (leader) {
            uint64_t *const fb = &kv_full[slot];
            // one 128-row box, or 16 sink rows + a 112-row band box (fused first block)
            ptx::mbar_arrive_expect_tx(fb, kBlockKeys * 128 * C::kHalves);
            uint8_t *dst = sKV + slot * C::kSlotBytes;
            for (int h = 0; h < C::kHalves; ++h) {
              if (b.sink) {
                ptx::tma_load_3d(dst + h * C::kSlotHalfBytes, kv ? &p.tm_vs : &p.tm_ks,
                                 fb, h * 64, 0, f.kvh);
                ptx::tma_load_3d(dst + h * C::kSlotHalfBytes + kSinkRows * 128,
                                 kv ? &p.tm_vb : &p.tm_kb, fb, h * 64, b.kb, f.kvh);
              } else {
                ptx::tma_load_3d(dst + h * C::kSlotHalfBytes, kv ? &p.tm_v : &p.tm_k,
                                 fb, h * 64, b.kb, f.kvh);
              }
            }
            TRACE_PR(2 + kv, j);
          }
        }
      };
      // Item order on the ring: K0 V0 of item i go out as soon as their slots free up;
      // Q(i) (which waits for the previous item's last QK^T) follows; the next item's Q
      // tiles are prefetched into L2 one item ahead so the Q load at the item boundary is
      // an L2 hit rather than an HBM round trip.
      // Item source: this CTA's own list, then entries of the shared tail fetched from a
      // global counter (the next one is fetched while the current item loads).
      const uint32_t own0 = p.offsets[blockIdx.x], own1 = p.offsets[blockIdx.x + 1];
      // Tail counter reset in-kernel (no memset launch before the kernel): CTA 0 swaps in
      // {this launch's epoch, count 0} with an atomic at L2.
#ifndef TA_QUEUE_MEMSET
      if (blockIdx.x == 0 && leader)
        atomicExch(reinterpret_cast<unsigned long long *>(p.queue), (unsigned long long)p.epoch << 32);
#endif
      const int leader_lane = __ffs(__ballot_sync(0xffffffffu, leader)) - 1;
      auto fetch = [&](uint32_t k) -> int {  // item index of this CTA's k-th item, -1 = none
        if (own0 + k < own1) return (int)(own0 + k);
        uint32_t t = 0;
        if (leader) {
          // queue word = epoch << 32 | count.  A ticket is valid only if it carries this
          // launch's epoch, i.e. CTA 0's reset came first (normally long before: a CTA
          // reaches the tail after its own list); an increment that hit the previous
          // launch's word is overwritten by the reset and retried.
#ifdef TA_QUEUE_MEMSET  // (experiment) host memset before the launch, plain 32-bit ticket
          t = atomicAdd(p.queue, 1u);
#else
          unsigned long long v = atomicAdd(reinterpret_cast<unsigned long long *>(p.queue), 1ull);
          if (__builtin_expect((v >> 32) != p.epoch, 0)) v = stale_ticket_retry(p.queue, p.epoch);
          t = (uint32_t)v;
#endif
        }
        t = __shfl_sync(0xffffffffu, t, leader_lane);
        return t < (uint32_t)p.n_tail ? p.tail0 + (int)t : -1;
      };
      int next = fetch(0);
      for (;; ++nitem) {
        const int cur = next;
        const uint32_t rslot = nitem % kItemRing;
        if (!TA_RING_NOEMPTY) WS(0, ptx::mbar_wait_lazy(&item_empty[rslot], ((nitem / kItemRing) & 1u) ^ 1u));
        if (leader) {
          item_ring[rslot] = cur;
          ptx::mbar_arrive(&item_full[rslot]);  // release: the entry is visible to the waiters
        }
        if (cur < 0) break;
        ItemInfo f;
        item_info(p, p.items[cur], f);
        if (nitem == 0 && TA_COLD_START) {
          // Kernel start: every CTA's ring and Q tiles are empty and the data is in HBM, so
          // the first tile loads of all CTAs form one burst.  Only what the first QK^T needs
          // (Q, K0) goes out first; V0 and the rest of the ring follow once Q has landed,
          // which moves the first tensor work forward by the rest of the burst.
          load_q(f, nitem);
          load_kv(f, 0, 0, 1);
          WS(0, ptx::mbar_wait_lazy(q_full, 0u));
          load_kv(f, 0, 1, 2);
        } else {
          load_kv(f, 0);
          if (!TA_EXP_QONCE || nitem == 0) load_q(f, nitem);
        }
        // fetch the next entry only now: a tail fetch's atomic round trip overlaps this
        // item's loads instead of delaying them
        next = fetch(nitem + 1);
        if (leader && next >= 0) {
          ItemInfo fn;
          item_info(p, p.items[next], fn);
          for (int x = 0; x < 2; ++x)
            for (int h = 0; h < C::kHalves; ++h)
              ptx::tma_prefetch_l2_3d(&p.tm_q, h * 64, fn.r0 + x * p.tile_tokens, fn.kvh * p.group);
        }
        for (int j = 1; j < f.nb; ++j) load_kv(f, j);
      }
    }
    WS_DUMP(0, leader);
    __syncwarp();
  } else if (warp == kMmaWarp) {
    // ===================== MMA issuer (whole warp, one elected lane issues) ============
    const bool leader = ptx::elect_one();
    WS_DECL;
    {
#ifdef TA_TRACE
      uint32_t trc = 0;
#endif
      // TMEM columns: S_x at 128 x, O_x at 256 + 128 x
      const uint32_t qbase = ptx::smem_u32(sQ);
      const uint32_t kvbase = ptx::smem_u32(sKV);
      const uint32_t idesc_pv = ptx::idesc_bf16(128, D, 1);
      uint32_t seq = 0, nitem = 0;
      uint32_t pph[2] = {0, 0};
      // Descriptors are built once; per MMA only the 14-bit start-address field moves
      // (smem offsets < 256 KB, so adding (offset >> 4) to the descriptor never carries).
      uint64_t dq = ptx::sdesc_sw128(qbase, 16, 1024);
      uint64_t dkv = ptx::sdesc_sw128(kvbase, 16, 1024);
      uint64_t dkv_mn = ptx::sdesc_sw128(kvbase, C::kSlotHalfBytes, 1024);
      uint32_t tm = tmem_base();
      // Re-materialise the bases every iteration (an opaque asm "redefines" them): the
      // compiler would otherwise hoist all 32 per-k-step descriptors / TMEM addresses out
      // of the loop and spill them to local memory in this 72-register warp, putting
      // local-memory round trips between the waits and the MMA issues.
      auto opaque_bases = [&]() {
#if TA_MMA_REMAT
        asm volatile("" : "+l"(dq), "+l"(dkv), "+l"(dkv_mn), "+r"(tm));
#endif
      };
      // S_x[:, 0:ncols] = Q_x K_slot^T  (K-major A and B, 8 x K=16 steps over d)
      auto issue_qk = [&](int x, uint32_t kslot, const ItemInfo &fq, const Blk &b) {
        if (!leader) return;
        const uint64_t a0 = dq + (uint64_t)((x * C::kQTileBytes) >> 4);
        const uint64_t b0 = dkv + (uint64_t)((kslot * C::kSlotBytes) >> 4);
        const uint32_t idesc = ptx::idesc_bf16(128, tile_ncols(fq, b, x, p.tile_tokens), 0);
#pragma unroll
        for (int s = 0; s < D / 16; ++s) {
          const uint32_t qo = ((s >> 2) * C::kHalfBytes + (s & 3) * 32) >> 4;
          const uint32_t ko = ((s >> 2) * C::kSlotHalfBytes + (s & 3) * 32) >> 4;
          ptx::mma_ss(tm + 128u * x, a0 + qo, b0 + ko, idesc, s > 0 ? 1u : 0u);
        }
      };
      // O_x += P_x V_slot; P_x (bf16) lives in the S_x columns; V MN-major (d contiguous).
      // k-steps [s0, s1) of the block (keys 16 s .. 16 s + 15)
      auto issue_pv = [&](int x, uint32_t vslot, const ItemInfo &fq, const Blk &b, bool acc, int s0, int s1) {
        if (!leader) return;
        const uint64_t b0 = dkv_mn + (uint64_t)((vslot * C::kSlotBytes) >> 4);
        const int ksteps = tile_ncols(fq, b, x, p.tile_tokens) / 16;
        const uint32_t pcol = tm + 128u * x;
        // P of keys [64h, 64h + 64) sits in TMEM columns [64h, 64h + 32) of S_x when two
        // threads share a row (each writes over its own S columns), else in [0, 64).
#pragma unroll
        for (int s = s0; s < s1; ++s)
          if (s < ksteps)
            ptx::mma_ts(tm + 256u + 128u * x,
                        pcol + (s / (8 / kHPR)) * 64 + (s % (8 / kHPR)) * 8,
                        b0 + (uint64_t)(s * (2048 >> 4)), idesc_pv, (acc || s > 0) ? 1u : 0u);
      };
      auto commit = [&](uint64_t *bar) {
        if (leader) ptx::tc_commit(bar);
      };
      // The MMA stream is flat across items: [PV_A(j), QK_A(j+1), PV_B(j), QK_B(j+1)] where
      // block j+1 may be block 0 of the next item, so a new item's first QK^T overlaps the
      // previous item's last softmax instead of draining the pipeline.
      const int idx0 = take_item(0);
      if (idx0 >= 0) {
        ItemInfo f;
        item_info(p, p.items[idx0], f);
        uint32_t ii = 0;  // this CTA's item counter
        int j = 0;
        WS(0, MMA_WAIT(q_full, nitem & 1u));
        ptx::tc_fence_after();
        TRACE_MM(16, nitem);
        Blk b = block_info(f, 0);
        uint32_t kslot, kph, vslot, vph;
        ring_pos(seq, C::kStages, kslot, kph);
        MMA_WAIT(&kv_full[kslot], kph);
        ptx::tc_fence_after();
        WS(8, issue_qk(0, kslot, f, b));
        WS(10, commit(&s_full[0]));
        WS(8, issue_qk(1, kslot, f, b));
        WS(10, commit(&s_full[1]));
        WS(10, commit(&kv_empty[kslot]));
        if (f.nb == 1) commit(q_empty);  // Q tiles are free after the item's last QK^T
        while (true) {
          opaque_bases();
          ring_pos(seq + 1, C::kStages, vslot, vph);
          TRACE_MM(9, j);
          WS(1, MMA_WAIT(&kv_full[vslot], vph));
          for (int w = 0; w < TA_EXTRA_WAITS; ++w) MMA_WAIT(&kv_full[vslot], vph);
          TRACE_MM(17, j);
          // next block in the flat stream (same item j+1, or block 0 of the next item)
          const bool last = (j + 1 == f.nb);
          const int nidx = last ? take_item(ii + 1) : 0;  // the next queue entry
          const bool more = !last || nidx >= 0;
          ItemInfo f1 = f;
          int j1 = j + 1;
          if (last && more) {
            WS(11, item_info(p, p.items[nidx], f1));
            j1 = 0;
          }
          Blk b1 = b;
          uint32_t kslot1 = 0, kph1 = 0;
          if (more) {
            b1 = block_info(f1, j1);
            ring_pos(seq + 2, C::kStages, kslot1, kph1);
            // K of the next block is normally resident long before it is needed: wait for
            // it here, off the PV -> QK^T hand-off of tile A.
            if (TA_EARLY_K) MMA_WAIT(&kv_full[kslot1], kph1);
          }
          // ---- tile A: PV_A(j), then QK_A(next)
          TRACE_MM(8, j);
          spin_cycles(TA_DELAY_MMA);
          if (TA_PV_SPLIT) {
            WS(3, MMA_WAIT(&p_ready[0], pph[0]));
            pph[0] ^= 1u;
            ptx::tc_fence_after();
          }
          TRACE_MM(10, j);
          const uint32_t kitem = ii;  // item of block j
          if (j == 0 && kitem > 0) WS(5, MMA_WAIT(&o_free[0], (kitem - 1) & 1u));  // O_A drained
#ifdef TA_WAITSTAT
          if (j == 0) ++ws_acc[15];  // items
          ++ws_acc[14];              // block pairs
#endif
          bool qk_a_done = false;
          if (TA_EXP_QKEARLY && more) {  // timing probe: QK_A(next) before PV_A (overwrites P)
            if (last) {
              ++nitem;
              WS(0, MMA_WAIT(q_full, nitem & 1u));
            }
            WS(2, MMA_WAIT(&kv_full[kslot1], kph1));
            ptx::tc_fence_after();
            WS(8, issue_qk(0, kslot1, f1, b1));
            WS(10, commit(&s_full[0]));
            qk_a_done = true;
          }
          if (TA_PV_SPLIT) {
            WS(9, issue_pv(0, vslot, f, b, j > 0, 0, kSplit));  // keys 0..16 kSplit - 1 while the softmax finishes the rest
            WS(4, MMA_WAIT(&p_hi[0], pph[0] ^ 1u));
          } else {
            MMA_WAIT(&p_hi[0], pph[0]);
            pph[0] ^= 1u;
          }
          ptx::tc_fence_after();
          if (!TA_PV_SPLIT) issue_pv(0, vslot, f, b, j > 0, 0, kSplit);
          WS(9, issue_pv(0, vslot, f, b, j > 0, kSplit, 8));
          TRACE_MM(11, j);
          if (last) commit(&o_full[0]);
          if (more && !qk_a_done) {
            if (last) {  // the next item's Q tiles
              ++nitem;
              if (!TA_EXP_QONCE) WS(0, MMA_WAIT(q_full, nitem & 1u));
              TRACE_MM(16, nitem);
            }
            TRACE_MM(18, j);
            if (!TA_EARLY_K) WS(2, MMA_WAIT(&kv_full[kslot1], kph1));
            ptx::tc_fence_after();
            TRACE_MM(19, j);
            WS(8, issue_qk(0, kslot1, f1, b1));
            WS(10, commit(&s_full[0]));
            TRACE_MM(12, j);
          }
          // ---- tile B: PV_B(j), then QK_B(next)
          TRACE_MM(7, j);
          if (TA_PV_SPLIT) {
            WS(6, MMA_WAIT(&p_ready[1], pph[1]));
            pph[1] ^= 1u;
            ptx::tc_fence_after();
          }
          TRACE_MM(13, j);
          if (j == 0 && kitem > 0) WS(5, MMA_WAIT(&o_free[1], (kitem - 1) & 1u));  // O_B drained
          bool qk_b_done = false;
          if (TA_EXP_QKEARLY && more) {  // timing probe (see tile A)
            ptx::tc_fence_after();
            WS(8, issue_qk(1, kslot1, f1, b1));
            WS(10, commit(&s_full[1]));
            qk_b_done = true;
          }
          if (TA_PV_SPLIT) {
            WS(9, issue_pv(1, vslot, f, b, j > 0, 0, kSplit));  // keys 0..16 kSplit - 1 while the softmax finishes the rest
            WS(7, MMA_WAIT(&p_hi[1], pph[1] ^ 1u));
          } else {
            MMA_WAIT(&p_hi[1], pph[1]);
            pph[1] ^= 1u;
          }
          ptx::tc_fence_after();
          if (!TA_PV_SPLIT) issue_pv(1, vslot, f, b, j > 0, 0, kSplit);
          WS(9, issue_pv(1, vslot, f, b, j > 0, kSplit, 8));
          TRACE_MM(14, j);
          if (last) commit(&o_full[1]);
          WS(10, commit(&kv_empty[vslot]));
          seq += 2;
          if (!more) break;
          if (!qk_b_done) {
            WS(8, issue_qk(1, kslot1, f1, b1));
            WS(10, commit(&s_full[1]));
          }
          TRACE_MM(15, j);
          WS(10, commit(&kv_empty[kslot1]));
          if (j1 + 1 == f1.nb) commit(q_empty);  // last QK^T of that item issued
          if (last) ++ii;
          f = f1;
          j = j1;
          b = b1;
        }
      }
    }
    WS_DUMP(1, leader);
    __syncwarp();
  } else if (warp >= kSmWarp0 && warp < kSmWarp0 + kSoftmaxWarps) {
    // ===================== softmax / epilogue =====================
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegSoftmax) : "memory");
    WS_DECL;
    const int x = (warp - kSmWarp0) / (4 * kHPR);    // Q tile
    const int hc = ((warp - kSmWarp0) / 4) % kHPR;   // column part: S columns [kNCol hc, kNCol (hc + 1))
    const int wq = warp % 4;            // TMEM lane quarter
    const int r = wq * 32 + lane;       // packed row = TMEM lane
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    const uint32_t tmem = tmem_base();
    const uint32_t tS = tmem + x * 128 + hc * 64 + lane_off;  // own S columns; own P columns
    const uint32_t tO = tmem + 256 + x * 128 + hc * (D / kHPR) + lane_off;  // own O columns
    const int T = p.tile_tokens;
    const bool row_in_tile = r < p.group * T;
    const int toff = row_in_tile ? r % T : 0;
    const float sc = p.scale_log2;
    const int c0 = hc * kNCol;  // first S column of this thread
    // shared-space addresses (explicit st.shared / ld.shared, not generic accesses)
    const uint32_t my_max_s = ptx::smem_u32(red_max + (x * 2 * 2 + hc) * kTileRows + r);
    const uint32_t peer_max_s = ptx::smem_u32(red_max + (x * 2 * 2 + (1 - hc)) * kTileRows + r);
    uint32_t sph = 0, ecount = 0, kitem_sm = 0;
    // Softmax -> MMA / epilogue hand-offs: one arrival per warp (TA_WARP_ARRIVE; the
    // warp-collective tcgen05.wait::st / __syncwarp order the other lanes' TMEM and shared
    // stores before lane 0's release-arrive) instead of 32 serialised same-address arrivals.
    auto sm_arrive = [&](uint64_t *bar) {
      if (TA_WARP_ARRIVE) {
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(bar);
      } else {
        ptx::mbar_arrive(bar);
      }
    };
    auto sm_arrive_state = [&](uint64_t *bar) -> uint64_t {
      if (TA_WARP_ARRIVE) {
        __syncwarp();
        uint64_t st = 0;
        if (lane == 0) st = ptx::mbar_arrive_state(bar);
        return __shfl_sync(0xffffffffu, st, 0);
      }
      return ptx::mbar_arrive_state(bar);
    };
#ifdef TA_TRACE
    uint32_t trc = 0;
#endif
    for (uint32_t ii = 0;; ++ii) {
      const int idx = take_item(ii);
      if (idx < 0) break;
      ItemInfo f;
      item_info(p, p.items[idx], f);
      const int tok = f.r0 + x * T + toff;     // query row i of this thread
      const bool last_row = tok >= p.n - p.last;
      float m_run = -INFINITY;  // reference max, log2 units of scaled scores
      float l_run = 0.f;        // running sum of 2^(x - m_run) over this thread's columns
#ifdef TA_COUNT
      uint32_t n_adm = 0, n_cmp = 0;
#endif
      for (int j = 0; j < f.nb; ++j) {
        const Blk b = block_info(f, j);
        // Kept columns of row i in this block: [a_lo, a_hi] U [b_lo, b_hi]   (reading R1)
        //   STREAM fused block 0: sink cols j < si, j <= i, then band cols
        //   STREAM sink block    : j < si, j <= i
        //   STREAM band block    : i - sl < j <= i (band keys are >= si)
        //   LASTQ                : triangle predicate within the chunk
        //   DENSE                : j <= i
        // Sink and band columns never cover the same key twice.
        const int khi = b.kb + b.nk - 1;  // last key loaded in the slot
        int a_lo = 0, a_hi = -1, b_lo, b_hi;
        if (f.kind == kStream) {
          if (b.sinkblk) {
            b_lo = b.kb;
            b_hi = min(min(p.si - 1, tok), khi);
          } else {
            b_lo = max(tok - p.sl + 1, b.kb);
            b_hi = min(tok, khi);
          }
          if (b.sink) a_hi = min(p.si, tok + 1) - 1;
        } else if (f.kind == kLastQ) {
          if (!last_row) {
            a_lo = max(f.kb0, b.kb);
            a_hi = min(min(p.si - 1, tok), min(f.ke0 - 1, khi));
          }
          b_lo = max(b.kb, last_row ? f.kb0 : max(f.kb0, tok - p.sl + 1));
          b_hi = min(min(f.ke0 - 1, tok), khi);
        } else {
          b_lo = b.kb;
          b_hi = min(tok, khi);
        }
        // keys -> columns of this thread's half
        if (f.kind != kStream || !b.sink) {
          a_lo -= b.kb;
          a_hi -= b.kb;
        }
        b_lo += b.sink - b.kb - c0;
        b_hi += b.sink - b.kb - c0;
        a_lo -= c0;
        a_hi -= c0;
        norm_iv(a_lo, a_hi);
        norm_iv(b_lo, b_hi);
#ifdef TA_COUNT
        {  // admitted keys of this row in the block (its kept-column intervals within the
           // computed columns) and the S columns the MMA computed for it
          const int lim = tile_ncols(f, b, x, T) - 1 - c0;
          auto span = [&](int lo, int hi) { lo = max(lo, 0); hi = min(hi, lim); return hi >= lo ? hi - lo + 1 : 0; };
          n_adm += span(a_lo, a_hi) + span(b_lo, b_hi);
          n_cmp += tile_ncols(f, b, x, T);
        }
#endif
        // All kNCol columns are processed every block (columns >= ncols are masked): no
        // data-dependent branches inside the row loop.
        constexpr int L = kNCol - 1;
        const bool full = (b_lo <= 0 && b_hi >= L) || (a_lo <= 0 && a_hi >= L) ||
                          (a_lo <= 0 && b_lo <= a_hi + 1 && b_hi >= L);
        const bool warp_full = __all_sync(0xffffffffu, full);

#if TA_SM_WAIT == 1
        while (!ptx::mbar_try_wait_hint(&s_full[x], sph, 1000000u)) {
        }
#else
        WS(0, ptx::mbar_wait(&s_full[x], sph));
#endif
        sph ^= 1u;
        ptx::tc_fence_after();
        TRACE_SM(20, j);
        TRACE_SMW(20, j);
        // The block body is compiled twice: for full-width blocks (8 16-column chunks) and
        // for short ones (<= 80 S columns: the diagonal block of a STREAM item at P = 64,
        // every other dense diagonal block), whose exponentials stop at the computed columns
        // with no runtime branch in the exponential loop (TA_SHORT_BODY).
        auto block_body = [&](auto nch_tag) {
        constexpr int kCh = decltype(nch_tag)::value;
        uint32_t s[kNCol];
        // 16-column groups this tile computes (tile_ncols; kHPR == 1): the rest of the S
        // columns hold no scores of this block and are skipped (they are masked anyway).
        const int nch = (kHPR == 1 && TA_TILE_TRIM == 1) ? tile_ncols(f, b, x, T) / 16
                        : (kHPR == 1 && TA_SKIP_RAGGED) ? b.ncols / 16 : kCh;
        // Two halves: the second TMEM load is in flight while the first half is masked.
        if (TA_TMEM_WIDE && kHPR == 1 && TA_TILE_TRIM == 0) {  // 32-column loads
#pragma unroll
          for (int c = 0; c < 2; ++c) ptx::tmem_ld32(tS + c * 32, s + c * 32);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int c = 2; c < 4; ++c)
            if (32 * c < 16 * kCh) ptx::tmem_ld32(tS + c * 32, s + c * 32);
        } else {
#pragma unroll
          for (int c = 0; c < kNCol / 32; ++c)
            if (c < nch) ptx::tmem_ld16(tS + c * 16, *reinterpret_cast<uint32_t(*)[16]>(s + c * 16), 0);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int c = kNCol / 32; c < kNCol / 16; ++c)
            if (c < nch) ptx::tmem_ld16(tS + c * 16, *reinterpret_cast<uint32_t(*)[16]>(s + c * 16), 0);
        }
        TRACE_SM(24, j);
#pragma unroll
        for (int c = 0; c < kNCol / 32; ++c) {
          if (c == kNCol / 64) ptx::tmem_wait_ld();
          if (!TA_EXP_NOMASK && !warp_full && 2 * c < nch) {
            // kept-column bitmask of chunk c: [a_lo, a_hi] U [b_lo, b_hi] intersected with
            // [32c, 32c + 31]
            const uint32_t m32 = iv_bits(a_lo - 32 * c, a_hi - 32 * c) | iv_bits(b_lo - 32 * c, b_hi - 32 * c);
            // TA_MASK_VOTE: skip the selects of a 32-column chunk every row of the warp keeps
            if (!TA_MASK_VOTE || __any_sync(0xffffffffu, m32 != 0xffffffffu)) {
#pragma unroll
              for (int e = 0; e < 32; ++e)
                s[c * 32 + e] = (m32 & (1u << e)) ? s[c * 32 + e] : 0xff800000u;  // -inf
            }
          }
        }
        // raw row max over this half (scale > 0 commutes with max), then over the row
        float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
        for (int e = 0; e < kNCol; e += 8) {
          if (e >= 16 * nch) break;
          mx0 = max3(mx0, __uint_as_float(s[e]), __uint_as_float(s[e + 1]));
          mx1 = max3(mx1, __uint_as_float(s[e + 2]), __uint_as_float(s[e + 3]));
          mx2 = max3(mx2, __uint_as_float(s[e + 4]), __uint_as_float(s[e + 5]));
          mx3 = max3(mx3, __uint_as_float(s[e + 6]), __uint_as_float(s[e + 7]));
        }
        float mx = max3(mx0, mx1, fmaxf(mx2, mx3));
        if (kHPR == 2) {  // row max over both column halves
          sts_f32(my_max_s + (j & 1) * 2 * kTileRows * 4, mx);
          asm volatile("bar.sync %0, %1;" ::"r"(1 + x), "r"(8 * 32) : "memory");
          mx = fmaxf(mx, lds_f32(peer_max_s + (j & 1) * 2 * kTileRows * 4));
        }
        const float m_new = fmaxf(m_run, mx * sc);
        TRACE_SM(25, j);
        const bool need = m_new > m_run + kRescaleThreshold;
        if (__any_sync(0xffffffffu, need)) {
          const float alpha = need ? ptx::ex2(m_run - m_new) : 1.f;
          if (need) m_run = m_new;
          l_run *= alpha;
          if (j > 0) {
            // O_x holds exactly blocks < j: S_x(j) completing implies PV_x(j-1) completed.
#pragma unroll 1
            for (int c = 0; c < D / (16 * kHPR); ++c) {
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
        // Ping-pong with the other tile: the exp phases (MUFU-heavy) of the two Q tiles
        // alternate, so each runs at full SMSP throughput while the tensor core works on
        // the other tile.
        if (kPingPong) ptx::mbar_wait(&exp_turn[x], (ecount & 1u) ^ (x == 0 ? 1u : 0u));
        spin_cycles(TA_DELAY_SM);
        const uint64_t sc2 = f2pack(sc, sc);
        uint64_t nref2 = f2pack(-ref, -ref);
#if TA_SUM_ROUNDED == 4
        float lsa = 0.f, lsb = 0.f, lsc = 0.f, lsd = 0.f;  // FHADD partial row sums
#else
        uint64_t l2a = 0, l2b = 0;  // packed partial row sums (FADD2)
#endif
        uint32_t pkw[16];           // bf16 P pairs of one (TA_TMEM_WIDE: two) 16-key chunks
#pragma unroll
        for (int c = 0; c < kNCol / 16; ++c) {
          if (c >= nch) {
            if (kHPR == 1 && c == kSplit - 1 && TA_PV_SPLIT) {  // keep the p_ready hand-off when the block is short
              ptx::tmem_wait_st();
              ptx::tc_fence_before();
              sm_arrive(&p_ready[x]);
            }
            continue;
          }
          uint32_t *pk = pkw + (TA_TMEM_WIDE ? (c & 1) * 8 : 0);
#pragma unroll
          for (int e = 0; e < 16; e += 2) {
            const int col = c * 16 + e;
            // x = s * scale * log2(e) - ref  for a register pair (FFMA2)
            const uint64_t xx = ffma2(u2pack(s[col], s[col + 1]), sc2, nref2);
            float x0, x1, p0, p1;
            f2unpack(xx, x0, x1);
            if ((kPolyPairs >> ((col >> 1) & 7)) & 1) {
              exp2_poly2(x0, x1, p0, p1);   // FMA pipe
            } else {
              p0 = ptx::ex2(x0);            // MUFU
              p1 = ptx::ex2(x1);
            }
#if TA_SUM_ROUNDED == 3
            // P truncated to bf16 on the ALU pipe (LOP3 x2 + PRMT instead of F2FP); the row
            // sum adds exactly the values the PV MMA consumes (exact normalisation).
            const uint32_t t0 = hi16(__float_as_uint(p0)), t1 = hi16(__float_as_uint(p1));
            pk[e / 2] = prmt_hi(__float_as_uint(p0), __float_as_uint(p1));
            const uint64_t pr = u2pack(t0, t1);
#elif TA_SUM_ROUNDED == 4
            pk[e / 2] = ptx::pack_bf16(p0, p1);
            // mixed-precision adds (FHADD.BF16) of the two rounded halves
#if TA_FHADD_ACC == 2
            sum_bf16_lo(lsa, pk[e / 2]);
            sum_bf16_hi(lsb, pk[e / 2]);
#else
            if (e & 2) {
              sum_bf16_lo(lsa, pk[e / 2]);
              sum_bf16_hi(lsb, pk[e / 2]);
            } else {
              sum_bf16_lo(lsc, pk[e / 2]);
              sum_bf16_hi(lsd, pk[e / 2]);
            }
#endif
#else
            pk[e / 2] = ptx::pack_bf16(p0, p1);
#if TA_SUM_ROUNDED == 1
            // row sum of the bf16-rounded P the PV MMA actually uses (exact normalisation)
            const uint64_t pr = u2pack(pk[e / 2] << 16, pk[e / 2] & 0xffff0000u);
#elif TA_SUM_ROUNDED == 2
            // the same with both unpacks forced onto the ALU pipe (PRMT + LOP3)
            const uint64_t pr = u2pack(lo16_up(pk[e / 2]), hi16(pk[e / 2]));
#else
            const uint64_t pr = f2pack(p0, p1);
#endif
#endif
#if TA_SUM_ROUNDED != 4
            if (e & 2)
              l2b = fadd2(l2b, pr);
            else
              l2a = fadd2(l2a, pr);
#endif
          }
          if (!TA_TMEM_WIDE)
            ptx::tmem_st8(tS + c * 8, pk);
          else if (c & 1)  // two chunks (32 keys) per 16-column store
            ptx::tmem_st16(tS + (c - 1) * 8, pkw);
          else if (c == kCh - 1)  // odd chunk count (short body): the last chunk alone
            ptx::tmem_st8(tS + c * 8, pk);
          if (kHPR == 1 && c == kSplit - 1 && TA_PV_SPLIT) {
            // keys 0..63 of P are in TMEM: the MMA can start PV on them right away
            ptx::tmem_wait_st();
            ptx::tc_fence_before();
#if TA_EXP_ORDER
            // The exponentials of keys 64..127 take their offset from the arrive's state
            // token, so ptxas cannot schedule them above the hand-off (it otherwise hoists
            // all 128 exponentials above the first TMEM store and p_ready fires at the end
            // of the row, leaving PV nothing to overlap).
            nref2 = ptx::after_token(nref2, sm_arrive_state(&p_ready[x]));
#else
            sm_arrive(&p_ready[x]);
#endif
          }
        }
        __syncwarp();
        if (kPingPong && lane == 0) ptx::mbar_arrive(&exp_turn[1 - x]);
        ++ecount;
        TRACE_SM(26, j);
        {
#if TA_SUM_ROUNDED == 4
          l_run += (lsa + lsb) + (lsc + lsd);
#else
          const uint64_t l2 = fadd2(l2a, l2b);
          float a0, a1;
          f2unpack(l2, a0, a1);
          l_run += a0 + a1;
#endif
        }
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        sm_arrive((kHPR == 2 && hc == 0) ? &p_ready[x] : &p_hi[x]);
        };
        const bool short_ok = TA_SHORT_BODY && kHPR == 1 && TA_TILE_TRIM == 0 && !TA_SKIP_RAGGED &&
                              (!TA_SHORT_STREAM_ONLY || f.kind == kStream);
        if (TA_SHORT4 && short_ok && b.ncols <= 64)
          block_body(std::integral_constant<int, 4>{});
        else if (short_ok && b.ncols <= 80)
          block_body(std::integral_constant<int, 5>{});
        else
          block_body(std::integral_constant<int, kNCol / 16>{});
        TRACE_SM(21, j);
        TRACE_SMW(21, j);
      }
      // ---------------- hand the item's row statistics to the epilogue warpgroup
      {
        // Back-pressure: publish item k only after the epilogue released item k-1, so
        // l_ready never runs two phases ahead of its waiter (single-block items).
        if (kitem_sm > 0) WS(1, ptx::mbar_wait(&o_free[x], (kitem_sm - 1) & 1u));
        const uint32_t par = kitem_sm & 1u;
        sts_f32(ptx::smem_u32(red_l + ((par * 2 + x) * 2 + hc) * kTileRows + r), l_run);
        if (kHPR == 1) sts_f32(ptx::smem_u32(red_l + ((par * 2 + x) * 2 + 1) * kTileRows + r), 0.f);
        if (hc == 0) sts_f32(ptx::smem_u32(red_m + (par * 2 + x) * kTileRows + r), m_run);
        sm_arrive(&l_ready[x]);
        ++kitem_sm;
#ifdef TA_COUNT
        if (row_in_tile && tok < p.n) {
          uint32_t *cnt = reinterpret_cast<uint32_t *>(p.trace) +
                          2 * ((int64_t)(f.kvh * p.group + r / T) * p.n + tok);
          atomicAdd(cnt, n_adm);
          atomicAdd(cnt + 1, n_cmp);
        }
#endif
      }
    }
    WS_DUMP(2 + x, lane == 0 && wq == 0 && hc == 0);
  } else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + kEpiWarps) {
    // ===================== epilogue warpgroup =====================
    WS_DECL;
    // O_x = O_x / l per row from TMEM -> bf16 global (STREAM / DENSE) or fp32 split-K
    // partial + LSE (LASTQ); then O_x's TMEM columns are released to the MMA issuer.
    const int eq = warp % 4;           // TMEM lane quarter
    const int x0 = kEpiWarps == 8 ? (warp - kEpiWarp0) / 4 : 0;  // first Q tile served
    const int r = eq * 32 + lane;      // packed row
    const uint32_t lane_off = (uint32_t)(eq * 32) << 16;
    const int T = p.tile_tokens;
    const bool row_in_tile = r < p.group * T;
    const int hoff = row_in_tile ? r / T : 0;
    const int toff = row_in_tile ? r % T : 0;
    uint32_t kitem = 0;
#ifdef TA_TRACE
    uint32_t trc = 0;
#endif
    for (;; ++kitem) {
      const int idx = take_item(kitem);
      if (idx < 0) break;
      ItemInfo f;
      item_info(p, p.items[idx], f);
      const uint32_t par = kitem & 1u;
      for (int x = x0; x < (kEpiWarps == 8 ? x0 + 1 : 2); ++x) {
        const uint32_t tO = tmem_base() + 256 + x * 128 + lane_off;
        const int tok = f.r0 + x * T + toff;
        const bool valid = row_in_tile && tok < p.n;
        TRACE_EP(30 + x, kitem);
        WS(0, ptx::mbar_wait_lazy(&l_ready[x], par));
        WS(1, ptx::mbar_wait_lazy(&o_full[x], par));
        ptx::tc_fence_after();
        TRACE_EP(32 + x, kitem);
        const float l_row = lds_f32(ptx::smem_u32(red_l + ((par * 2 + x) * 2 + 0) * kTileRows + r)) +
                            lds_f32(ptx::smem_u32(red_l + ((par * 2 + x) * 2 + 1) * kTileRows + r));
        const float m_row = lds_f32(ptx::smem_u32(red_m + (par * 2 + x) * kTileRows + r));
        const float inv = l_row > 0.f ? 1.f / l_row : 0.f;
        const float lse = l_row > 0.f ? (m_row + __log2f(l_row)) * kLn2 : -INFINITY;
        if (TA_EXP_NOEPI) {
        } else if (f.kind == kLastQ) {
          const int64_t slot =
              ((int64_t)f.kvh * p.n_last_pairs + (f.pair - p.p_last0)) * p.s_max + f.chunk;
          const int64_t prow = slot * (2 * kTileRows) + x * kTileRows + r;
          float *dst = p.part_o + prow * D;
#pragma unroll 1
          for (int c = 0; c < D / 16; ++c) {
            uint32_t ov[16];
            ptx::tmem_ld16(tO + c * 16, ov, 0);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 16; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * inv);
            st_global_v8(dst + c * 16, ov);
            st_global_v8(dst + c * 16 + 8, ov + 8);
          }
          p.part_lse[prow] = lse;
        } else {
          const int head = f.kvh * p.group + hoff;
          // O tile -> bf16 -> smem (128 rows x 64 columns per pass, 128B-swizzled like the Q
          // tile) -> one TMA tensor store of box {64, T, G}: the same GQA-packed box the Q
          // tile was loaded with, so rows beyond G*T or tokens >= N are clipped by TMA.
          const uint32_t stage_s = ptx::smem_u32(stage);
#pragma unroll 1
          for (int hb = 0; hb < D / 64; ++hb) {
            uint32_t pk[32];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              uint32_t ov[16];
              ptx::tmem_ld16(tO + hb * 64 + c * 16, ov, 0);
              ptx::tmem_wait_ld();
#if TA_EPI_FMUL2
              // O / l with packed FMUL2 (half the FMA-pipe issue of the scalar multiplies)
              const uint64_t inv2 = f2pack(inv, inv);
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                uint64_t o2 = u2pack(ov[2 * e], ov[2 * e + 1]);
                asm("mul.rn.f32x2 %0, %0, %1;" : "+l"(o2) : "l"(inv2));
                float a0, a1;
                f2unpack(o2, a0, a1);
                pk[c * 8 + e] = ptx::pack_bf16(a0, a1);
              }
#else
#pragma unroll
              for (int e = 0; e < 8; ++e)
                pk[c * 8 + e] = ptx::pack_bf16(__uint_as_float(ov[2 * e]) * inv,
                                               __uint_as_float(ov[2 * e + 1]) * inv);
#endif
            }
            TRACE_EP(40 + hb, kitem);
            // staging buffer free: the previous TMA store has finished reading it
            if (threadIdx.x == kEpiWarp0 * 32) WS(2, ptx::bulk_wait_read0());
            WS(3, asm volatile("bar.sync 5, 128;" ::: "memory"));
            TRACE_EP(42 + hb, kitem);
            {
              // swizzled row addresses recomputed here (an opaque copy of r): hoisted out of
              // the item loop they occupy 8 registers of this 80-register warpgroup (spills)
              int rr = r;
              asm volatile("" : "+r"(rr));
              const uint32_t row_s = stage_s + rr * 128;
#pragma unroll
              for (int pc = 0; pc < 8; ++pc)
                sts_v4(row_s + ((pc ^ (rr & 7)) << 4), pk[4 * pc], pk[4 * pc + 1], pk[4 * pc + 2],
                       pk[4 * pc + 3]);
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("bar.sync 5, 128;" ::: "memory");
            if (threadIdx.x == kEpiWarp0 * 32) {
              ptx::tma_store_3d(&p.tm_o, stage, hb * 64, f.r0 + x * T, f.kvh * p.group);
              // f2: the same staged tile to every extra destination (peer ranks' O)
              if (kMode == kOutExtra)
                for (int e = 0; e < p.n_ox; ++e)
                  ptx::tma_store_3d(&p.tm_ox[e], stage, hb * 64, f.r0 + x * T, f.kvh * p.group);
              ptx::bulk_commit();
            }
            if (kMode == kOutMulticast) {
              // f2 multicast: the staged half tile (128 rows x 128 B, 128B-swizzled) to the
              // multicast view, 16 B per lane, 8 lanes per contiguous row segment.
              const int pc = (threadIdx.x - kEpiWarp0 * 32) & 7;
#pragma unroll 1
              for (int rr = (threadIdx.x - kEpiWarp0 * 32) >> 3; rr < kTileRows; rr += 16) {
                const int tk = f.r0 + x * T + rr % T;
                if (rr < p.group * T && tk < p.n) {
                  uint32_t w0, w1, w2, w3;
                  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                               : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3)
                               : "r"(stage_s + rr * 128 + ((pc ^ (rr & 7)) << 4)));
                  __nv_bfloat16 *dst = reinterpret_cast<__nv_bfloat16 *>(p.mc_o) +
                                       (int64_t)(f.kvh * p.group + rr / T) * p.mc_sh + (int64_t)tk * p.mc_st +
                                       hb * 64 + pc * 8;
                  mc_st16(dst, w0, w1, w2, w3);
                }
              }
            }
            TRACE_EP(44 + hb, kitem);
          }
          if (valid && p.lse) p.lse[(int64_t)head * p.n + tok] = lse;
        }
        // O_x has been read: the next item's first PV_x may overwrite it
        TRACE_EP(34 + x, kitem);
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&o_free[x]);
      }
    }
    WS_DUMP(4, lane == 0 && warp == kEpiWarp0);
  }
  if (threadIdx.x == kEpiWarp0 * 32) ptx::bulk_wait0();  // epilogue TMA stores complete
  __syncthreads();
  // PDL: this CTA's work is issued; the merge grid may begin launching (its
  // griddepcontrol.wait still orders every read after this grid's completion).
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#ifdef TA_CTA_CLOCK
  if (threadIdx.x == 0) {
    p.trace[blockIdx.x] = (unsigned long long)(clock64() - cta_t0);
#ifdef TA_GT  // (+0.8 % cycles: the entry timestamp stays live in warp 0 all kernel long)
    unsigned long long g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    p.trace[256 + 2 * blockIdx.x] = cta_g0;  // globaltimer (ns) at CTA start / end
    p.trace[257 + 2 * blockIdx.x] = g1;
#endif
  }
#endif
  if (warp == kAllocWarp) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base(), 512);
  }
}

// LSE merge of the split-K partials of the last pairs (merge_output; readings
// R8/R18): per packed row, O = sum_c e^{LSE_c - M} O_c / sum_c e^{LSE_c - M} over the pair's
// chunks c, M = max_c LSE_c; a chunk with LSE = -inf has weight 0.  W warps share a row
// (chunks strided over the warps; W grows with the chunk count so that rows with many
// chunks -- small head shards, where ck is small -- still spread over the whole GPU),
// combined through shared memory.  Launched with PDL (griddepcontrol.wait first).
#ifndef TA_MERGE_U  // chunks whose loads a merge warp issues before using them
#define TA_MERGE_U 4
#endif
template <int D, int W>
__global__ void __launch_bounds__(256) merge_kernel(const __grid_constant__ AttnParams p) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  constexpr int E = D / 32;
  constexpr int RPB = 8 / W;  // rows per block
  __shared__ float s_max[8], s_w[8];
  __shared__ float s_acc[8][D];  // [warp][32 e + lane]: element pair order of the lane
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int sub = warp % W, rib = warp / W;
  const int rows = 2 * kTileRows;
  const int64_t gr = (int64_t)blockIdx.x * RPB + rib;  // (kvh, last pair, packed row) linear
  const int64_t per_kvh = (int64_t)p.n_last_pairs * rows;
  const int kvh = (int)(gr / per_kvh);
  const int rem = (int)(gr % per_kvh);
  const int lp = rem / rows, rr = rem % rows;
  const int x = rr / kTileRows, r = rr % kTileRows;
  const int T = p.tile_tokens;
  const int pair = p.p_last0 + lp;
  const int tok = pair * p.pair_tokens + x * T + r % T;
  // rows without output still take part in the block barriers
  bool live = kvh < p.hq / p.group && r < p.group * T && tok < p.n &&
              !(p.last_only && tok < p.n - p.last);
  const int nch = live ? (int)p.span_pieces[(int64_t)kvh * p.n_last_pairs + lp] : 0;
  const int64_t slot0 = ((int64_t)kvh * p.n_last_pairs + lp) * p.s_max;
  float mx = -INFINITY;
  for (int c = sub + W * lane; c < nch; c += 32 * W) mx = fmaxf(mx, p.part_lse[(slot0 + c) * rows + rr]);
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (W > 1) {
    if (lane == 0) s_max[warp] = mx;
    __syncthreads();
#pragma unroll
    for (int w = 0; w < W; ++w) mx = fmaxf(mx, s_max[rib * W + w]);
  }
  // lane owns the element pairs (2 lane + 64 q, 2 lane + 64 q + 1), q < E / 2
  float acc[E];
#pragma unroll
  for (int e = 0; e < E; ++e) acc[e] = 0.f;
  float wsum = 0.f;
  // U chunks per step with all their loads issued first (latency-bound loop).
  constexpr int U = TA_MERGE_U;
  for (int c0 = sub; c0 < nch; c0 += U * W) {
    float lcs[U], vv[U][E];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = c0 + u * W;
      lcs[u] = -INFINITY;
      if (c < nch) {
        lcs[u] = p.part_lse[(slot0 + c) * rows + rr];
        const float2 *src = reinterpret_cast<const float2 *>(p.part_o + ((slot0 + c) * rows + rr) * D);
#pragma unroll
        for (int q = 0; q < E / 2; ++q) {
          const float2 t = src[lane + 32 * q];
          vv[u][2 * q] = t.x;
          vv[u][2 * q + 1] = t.y;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (lcs[u] == -INFINITY) continue;  // empty chunk: weight 0, never exp(-inf - -inf)
      const float w = __expf(lcs[u] - mx);
      wsum += w;
#pragma unroll
      for (int e = 0; e < E; ++e) acc[e] += w * vv[u][e];
    }
  }
  if (W > 1) {
#pragma unroll
    for (int e = 0; e < E; ++e) s_acc[warp][32 * e + lane] = acc[e];
    if (lane == 0) s_w[warp] = wsum;
    __syncthreads();
    if (sub != 0) return;
    wsum = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) acc[e] = 0.f;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      wsum += s_w[rib * W + w];
#pragma unroll
      for (int e = 0; e < E; ++e) acc[e] += s_acc[rib * W + w][32 * e + lane];
    }
  }
  if (!live) return;
  const int head = kvh * p.group + r / T;
  const float inv = wsum > 0.f ? 1.f / wsum : 0.f;
  const int orow = tok - p.o_row0;
  uint32_t ov[E / 2];
#pragma unroll
  for (int q = 0; q < E / 2; ++q) ov[q] = ptx::pack_bf16(acc[2 * q] * inv, acc[2 * q + 1] * inv);
  uint32_t *dst = reinterpret_cast<uint32_t *>(reinterpret_cast<__nv_bfloat16 *>(p.o) +
                                               (int64_t)head * p.o_sh + (int64_t)orow * p.o_st);
#pragma unroll
  for (int q = 0; q < E / 2; ++q) dst[lane + 32 * q] = ov[q];
  for (int x2 = 0; x2 < p.n_ox; ++x2) {  // f2: extra destinations
    uint32_t *d2 = reinterpret_cast<uint32_t *>(reinterpret_cast<__nv_bfloat16 *>(p.ox[x2]) +
                                                (int64_t)head * p.ox_sh[x2] + (int64_t)orow * p.ox_st[x2]);
#pragma unroll
    for (int q = 0; q < E / 2; ++q) d2[lane + 32 * q] = ov[q];
  }
  if (p.mc_o) {  // f2 multicast view
    uint32_t *d2 = reinterpret_cast<uint32_t *>(reinterpret_cast<__nv_bfloat16 *>(p.mc_o) +
                                                (int64_t)head * p.mc_sh + (int64_t)orow * p.mc_st);
#pragma unroll
    for (int q = 0; q < E / 2; ++q) mc_st4(d2 + lane + 32 * q, ov[q]);
  }
  if (lane == 0 && p.lse)
    p.lse[(int64_t)head * (p.n - p.o_row0) + orow] = wsum > 0.f ? mx + __logf(wsum) : -INFINITY;
}

}  // namespace

size_t attention_smem_bytes(int head_dim) {
  return head_dim == 128 ? Cfg<128>::kSmem : Cfg<64>::kSmem;
}

template <int D, int M>
static cudaError_t launch_attention_t(const AttnParams &p, int num_ctas, cudaStream_t s) {
  // The dynamic shared-memory opt-in is per device (context): remember it per device id.
  static std::atomic<uint64_t> attr_set{0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = dev < 64 ? (1ull << dev) : 0ull;
  if (!bit || !(attr_set.load(std::memory_order_acquire) & bit)) {
    e = cudaFuncSetAttribute(attn_kernel<D, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<D>::kSmem);
    if (e != cudaSuccess) return e;
    attr_set.fetch_or(bit, std::memory_order_acq_rel);
  }
  attn_kernel<D, M><<<num_ctas, kThreads, Cfg<D>::kSmem, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_attention(const AttnParams &p, int head_dim, int num_ctas, cudaStream_t s) {
  if (p.mc_o)
    return head_dim == 128 ? launch_attention_t<128, kOutMulticast>(p, num_ctas, s)
                           : launch_attention_t<64, kOutMulticast>(p, num_ctas, s);
  if (p.n_ox > 0)
    return head_dim == 128 ? launch_attention_t<128, kOutExtra>(p, num_ctas, s)
                           : launch_attention_t<64, kOutExtra>(p, num_ctas, s);
  return head_dim == 128 ? launch_attention_t<128, kOutSingle>(p, num_ctas, s)
                         : launch_attention_t<64, kOutSingle>(p, num_ctas, s);
}

// Warps per merged row: enough that the split-K chunks of a row (s_max <= 8 at C3 on one
// GPU, up to 64-128 on an 8-way head shard) spread over the whole GPU.
template <int D>
static cudaError_t launch_merge_t(const AttnParams &p, int64_t rows, cudaLaunchConfig_t &cfg) {
  static const int forced = [] {  // TA_MERGE_W=1|2|4|8: experiment override
    const char *e = getenv("TA_MERGE_W");
    return e ? atoi(e) : 0;
  }();
  // measured (scripts/merge_w.py): C3 s_max 11: W = 1 12.8 us, 2 15.6, 4 17.0; 8-way C3
  // s_max 80: W = 8 12.5 us, 4 14.1, 1 24.4; 8-way C2 s_max 38: W = 8 8.4 us, 4 9.7
  const int w = forced ? forced : p.s_max <= 16 ? 1 : p.s_max <= 24 ? 4 : 8;
  const int64_t rpb = 8 / w;
  cfg.gridDim = dim3((unsigned)((rows + rpb - 1) / rpb));
  switch (w) {
    case 1: return cudaLaunchKernelEx(&cfg, merge_kernel<D, 1>, p);
    case 2: return cudaLaunchKernelEx(&cfg, merge_kernel<D, 2>, p);
    case 4: return cudaLaunchKernelEx(&cfg, merge_kernel<D, 4>, p);
    default: return cudaLaunchKernelEx(&cfg, merge_kernel<D, 8>, p);
  }
}

cudaError_t launch_merge(const AttnParams &p, int head_dim, int hkv, cudaStream_t s, bool pdl) {
  const int64_t rows = (int64_t)hkv * p.n_last_pairs * 2 * kTileRows;
  if (rows == 0) return cudaSuccess;
  // Programmatic dependent launch (merge_output follows the split-K pass):
  // the merge grid is launched while the attention grid drains.
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return head_dim == 128 ? launch_merge_t<128>(p, rows, cfg) : launch_merge_t<64>(p, rows, cfg);
}

}  // namespace ta
