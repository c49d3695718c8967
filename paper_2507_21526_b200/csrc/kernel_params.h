// kernel_params.h -- parameter block shared by the host launcher and the sm_100a kernels.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "schedule.h"

namespace ta {

constexpr int kMaxExtraOut = 7;  // TA_MAX_EXTRA_OUT

// Passed by value as a __grid_constant__ kernel parameter; the TMA descriptors
// must live in param space so cp.async.bulk.tensor can take their address.
struct alignas(64) AttnParams {
  CUtensorMap tm_q;  // Q [Hq][N][d]:   dims {d, N, Hq},  box {64, T, G}
  CUtensorMap tm_k;  // K [Hkv][N][d]:  dims {d, N, Hkv}, box {64, 128, 1}
  CUtensorMap tm_v;  // V, same as K
  CUtensorMap tm_ks; // K sink rows: box {64, 16, 1}
  CUtensorMap tm_vs; // V sink rows
  CUtensorMap tm_kb; // K band rows of a fused first block: box {64, 112, 1}
  CUtensorMap tm_vb; // V, same
  CUtensorMap tm_o;  // O [Hq][N][d] (bf16 output, epilogue TMA store): box {64, T, G}
  void *o;           // bf16 O [Hq][N][d] with element strides below
  int64_t o_sh, o_st;
  float *lse;        // optional [Hq][N - o_row0]
  float *part_o;     // split-K partials [slot][2*128 rows][d] fp32 (normalised O_c)
  float *part_lse;   // [slot][2*128 rows] fp32 natural-log LSE_c
  const Item *items;      // CTA c's own list items[offsets[c], offsets[c+1]), then the shared tail
  const uint32_t *offsets;
  const uint8_t *span_pieces;  // LASTQ pieces per (kvh, last pair) = merge chunk counts
  int tail0, n_tail;      // shared tail: items[tail0 .. tail0 + n_tail), fetched dynamically
  uint32_t *queue;        // 64-bit word {epoch (hi), next tail entry to fetch (lo)}
  uint32_t epoch;         // this launch's nonzero id: CTA 0 resets the word to {epoch, 0};
                          // tail tickets carrying another epoch are retried (no host memset)
  int n, hq, group, tile_tokens, pair_tokens;
  int si, sl, last, dense;
  int last_only;     // final-layer mode: the merge writes only rows >= N - last ...
  int o_row0;        // ... into O / lse whose row 0 is token o_row0 (0 otherwise)
  int p_last0, n_last_pairs, chunk_keys, s_max;
  float scale_log2;  // softmax_scale * log2(e)
  float scale;       // softmax_scale
  unsigned long long *trace;  // debug timeline (TA_TRACE builds only), else NULL
  int trace_cta;
  // f2: extra output destinations (triangle/dense_attn_prefill_multi), same layout as O
  int n_ox;
  void *ox[kMaxExtraOut];
  int64_t ox_sh[kMaxExtraOut], ox_st[kMaxExtraOut];
  CUtensorMap tm_ox[kMaxExtraOut];
  // f2 multicast: the same O view at a multicast virtual address (NVLS: one store reaches
  // every GPU bound to the multicast object); NULL = none.  Element strides as for o.
  void *mc_o;
  int64_t mc_sh, mc_st;
};

// Launchers (kernels.cu). Return the CUDA error of the launch.
cudaError_t launch_attention(const AttnParams &p, int head_dim, int num_ctas, cudaStream_t s);
cudaError_t launch_merge(const AttnParams &p, int head_dim, int hkv, cudaStream_t s, bool pdl);
size_t attention_smem_bytes(int head_dim);

}  // namespace ta
