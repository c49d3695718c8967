/* triattn.h -- C ABI v4 of the B200-native TriangleMix prefill-attention library.
 *
 * The library computes, for one prefill request (batch 1) and one attention
 * layer, the masked softmax attention of PAPER.md section 2.1
 *
 *     O = Softmax( Q K^T * scale - c (1 - M') ) V ,   c -> +inf  (reading R3)
 *
 * with M' chosen per layer by TriangleMix (section 2.4):
 *   dense layers    (layer <  tri_start):  M' = M, the causal mask;
 *   triangle layers (layer >= tri_start):  M' = M - M^middle, i.e. for 0-based
 *     query row i and key j <= i the pair is kept iff
 *         j < sink  or  i - j < window  or  i >= N - last_q
 *     (streaming section P:L120-131 + Last Q-K section; Middle Q-K
 *      section P:L163-172 skipped; index reading R1 in DESIGN.md).
 * The parameters are Algorithm 1's inputs (App. A.2):
 * Q, K, V in R^{N x d_h}; N_sink, N_window, N_last.  Grouped-query attention
 * ("generalizes naturally"): q head h reads kv head h / (Hq/Hkv)
 * (reading R13).
 *
 * Conventions (every function):
 *  - extern "C", never throws, never aborts, never prints.
 *  - Tensors are caller-owned CUDA DEVICE memory; the library keeps no pointer
 *    past the call.  Work is enqueued asynchronously on the caller's stream:
 *    keep buffers alive until the stream reaches that point.
 *  - Validation completes before anything is enqueued: on a non-OK return
 *    nothing was launched and O / lse / workspace are untouched.
 *  - Asynchronous device faults surface at the caller's next synchronisation.
 *  - Degenerate triangle parameters (sink+window+last_q >= N, last_q >= N,
 *    window >= N) are not errors: the result equals dense causal.
 *  - The library owns only host/device caches (schedules, TMA descriptors),
 *    keyed by device and problem signature, mutex-protected, freed by
 *    ta_release_caches().  Calls from different threads/streams are safe.
 *  - Same inputs + same SM count => bitwise-identical outputs.
 *  - Kernels run on the calling thread's CURRENT device (cudaGetDevice): every pointer
 *    and the stream must belong to it (the Python binding sets it from q's device).
 */
#ifndef TRIATTN_H_
#define TRIATTN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TA_ABI_VERSION 4  /* v2: last_q = 0 (StreamingMix), final-layer last-rows entry points;
                             v3: *_multi (f2); v4: ta_set_pdl, PDL-launched merge, multicast f2 */

/* Same type as the CUDA runtime's cudaStream_t (a duplicate identical typedef is
 * legal in C11/C++), so callers need no CUDA headers. NULL = legacy stream. */
typedef struct CUstream_st *cudaStream_t;

typedef enum {
  TA_OK = 0,
  TA_ERR_NULL_ARG = 1,       /* a required pointer is NULL                                      */
  TA_ERR_EMPTY_SEQUENCE = 2, /* seq_len == 0                       (SPEC EmptySequence S:L56)   */
  TA_ERR_SHAPE = 3,          /* heads < 1, Hq % Hkv != 0, seq_len < 0, stride too small
                                (SPEC ShapeError S:L168)                                        */
  TA_ERR_PARAMS = 4,         /* sink < 0, window < 1, last_q < 0 (< 1 for the last-rows
                                entry points), tri_start < 0, layer < 0, num_ctas < 1
                                (TriangleParams invariants S:L39-41)                            */
  TA_ERR_UNSUPPORTED = 5,    /* head_dim not in {64,128}; Hq/Hkv > 128; seq_len >= 2^31;
                                pointer not 16-byte aligned; stride*2 not a multiple of 16;
                                device is not sm_100                                             */
  TA_ERR_WORKSPACE = 6,      /* workspace NULL, too small, or not 256-byte aligned              */
  TA_ERR_CUDA = 7            /* CUDA error while enqueuing; detail in ta_last_error()          */
} ta_status;

/* bf16 tensor view [heads][tokens][head_dim], element strides, head_dim stride 1.
 * Head-major contiguous is stride_head = N*d, stride_token = d; token-major
 * [N][H][d] is stride_head = d, stride_token = H*d. */
typedef struct {
  const void *data;
  int64_t stride_head, stride_token;
} ta_in_tensor;
typedef struct {
  void *data;
  int64_t stride_head, stride_token;
} ta_out_tensor;

typedef struct {
  ta_in_tensor q, k, v;  /* q: Hq heads; k, v: Hkv heads; bf16; device pointers, caller-owned */
  ta_out_tensor o;       /* Hq heads, bf16, caller-owned, same shape as q                    */
  float *lse;            /* optional [Hq][seq_len] fp32 natural-log log-sum-exp of the kept
                            scores (Algorithm 1's "ln s + m"); NULL = not written     */
  int64_t seq_len;       /* N >= 1 tokens (batch = 1 prefill, reading R16)                    */
  int32_t num_q_heads;   /* Hq                                                                */
  int32_t num_kv_heads;  /* Hkv; q head h reads kv head h / (Hq/Hkv)                          */
  int32_t head_dim;      /* d in {64, 128}                                                    */
  float softmax_scale;   /* <= 0 -> 1/sqrt(head_dim)  ("1/sqrt(d)")                   */
} ta_problem;

/* Triangle shape (Algorithm 1 "Input triangle shape"): si, sl, last. */
typedef struct {
  int32_t sink;   /* si >= 0 sink key columns  j < si */
  int32_t window; /* sl >= 1 sliding-window keys  i - j < sl, incl. i */
  int32_t last_q; /* last >= 0 final query rows  i >= N - last;
                     0 = no Last Q-K section: the StreamingMix pattern of the paper's
                     baselines (reading R12)                          */
} ta_triangle;

/* Bytes of device workspace triangle_attn_prefill / dense_attn_prefill need: the split-K
 * partial outputs and their LSE for the Last-rows pass (triangle only) plus a
 * 256-byte block holding the fetch counter of the schedule's shared tail (every call; reset
 * inside the call's own kernel -- no separate memset -- so concurrent calls must use
 * different workspaces; its contents between calls need not be preserved).
 * tri == NULL -> dense.  Returns 0 on invalid arguments. */
size_t ta_workspace_size(const ta_problem *p, const ta_triangle *tri);

/* Triangle-shaped sparse causal attention of one deep layer,
 * Algorithm 1 re-designed for sm_100a: a static block schedule
 * of STREAM items (sink + sliding-window band per query tile, rows < N-last)
 * and LASTQ split-K items (rows >= N-last, all causal keys in pieces) assigned to
 * the persistent tcgen05/TMEM/TMA kernel's CTAs, plus a shared tail of items the
 * CTAs fetch dynamically when their own lists are done, then an LSE merge kernel
 * (P:L641-642).
 * ws: device workspace of >= ta_workspace_size(p, tri) bytes, 256-B aligned. */
ta_status triangle_attn_prefill(const ta_problem *p, const ta_triangle *tri, void *ws,
                                size_t ws_bytes, cudaStream_t stream);

/* Dense causal attention of one shallow layer; the same kernel
 * with DENSE items (keys [0, i] per row). ws: >= ta_workspace_size(p, NULL) bytes. */
ta_status dense_attn_prefill(const ta_problem *p, void *ws, size_t ws_bytes,
                             cudaStream_t stream);

/* Per-layer TriangleMix dispatch (reading R2): dense iff
 * layer < tri_start, else triangle with *tri. */
ta_status ta_layer_attn_prefill(int32_t layer, int32_t tri_start, const ta_problem *p,
                                const ta_triangle *tri, void *ws, size_t ws_bytes,
                                cudaStream_t stream);

/* ---- fused output replication ---------------------- *
 * Multi-GPU head sharding: rank r owns kv heads [r Hkv/P, (r+1) Hkv/P) and their q heads,
 * and every rank needs the full O [Hq][N][d] (the all-gather of 8(a) a7).  These calls run
 * the same kernels as triangle_attn_prefill / dense_attn_prefill, and the epilogue writes
 * each finished bf16 O tile, with the same TMA tensor store, to p->o AND to n_extra further
 * destinations extra_o[0..n_extra): typically this rank's head slice of the other ranks'
 * full-O buffers, mapped into this process (CUDA IPC / symmetric memory over NVLink), so
 * the gather overlaps the attention tile by tile instead of following it.  The LSE merge of
 * the last rows writes them to every destination as well.
 *   extra_o[e]: device pointer + strides of a bf16 [Hq][N][d] view (the same Hq heads
 *               and rows as p->o), 16-B aligned like p->o; caller-owned.
 *   0 <= n_extra <= TA_MAX_EXTRA_OUT; n_extra == 0 is exactly triangle_attn_prefill.
 * Visibility on the peers is the caller's business: after the call completes on this
 * rank's stream, a cross-rank barrier (e.g. symmetric-memory barrier or NCCL) must order
 * it before peers read their buffers.  Errors: TA_ERR_NULL_ARG (extra_o NULL with
 * n_extra > 0, or a NULL data pointer), TA_ERR_PARAMS (n_extra out of range),
 * TA_ERR_UNSUPPORTED (misaligned pointer / stride), as for p->o. */
#define TA_MAX_EXTRA_OUT 7
ta_status triangle_attn_prefill_multi(const ta_problem *p, const ta_triangle *tri,
                                      const ta_out_tensor *extra_o, int32_t n_extra, void *ws,
                                      size_t ws_bytes, cudaStream_t stream);
ta_status dense_attn_prefill_multi(const ta_problem *p, const ta_out_tensor *extra_o,
                                   int32_t n_extra, void *ws, size_t ws_bytes, cudaStream_t stream);

/* Multicast variant of f2 (NVLS, SURVEY 8(f) f2 as specified): the kernels additionally
 * write every finished O tile, and the merged last rows, with 16-byte multimem stores to
 * mc_o -- a [Hq][N][d] bf16 view (this rank's head slice) inside a buffer mapped at a
 * MULTICAST virtual address (cuMulticastCreate / cuMulticastBindMem / cuMemMap, or torch
 * symmetric memory's multicast_ptr) whose physical backing is every rank's full-O buffer.
 * Each tile leaves this GPU once and the NVSwitch delivers it to every bound GPU
 * (egress per rank = its O shard, vs (P - 1) x the shard for the unicast *_multi calls).
 * p->o is written as usual (it may be this rank's unicast view of the same buffer).
 *   mc_o: device multicast address + element strides; 16-B aligned, strides * 2 multiples
 *         of 16; caller-owned mapping (the library keeps no pointer past the call).
 * Visibility on the peers needs a cross-rank barrier after the call (as for *_multi).
 * Errors: TA_ERR_NULL_ARG (mc_o or its data NULL), TA_ERR_UNSUPPORTED (alignment), as for o.
 * The plain (non-multimem) store path is unaffected: separate kernel instantiation. */
ta_status triangle_attn_prefill_multicast(const ta_problem *p, const ta_triangle *tri,
                                          const ta_out_tensor *mc_o, void *ws, size_t ws_bytes,
                                          cudaStream_t stream);
ta_status dense_attn_prefill_multicast(const ta_problem *p, const ta_out_tensor *mc_o, void *ws,
                                       size_t ws_bytes, cudaStream_t stream);

/* ---- final layer: last query rows only ----------------------- *
 * "For the last layer, only the last r rows of the attention output are needed"
 * (TriangleMix section 2.4): O_last = Softmax(Q_last K^T * scale) V over ALL causal keys
 * of the last r = min(last_q, N) query rows, last_q >= 1.  Runs only the split-K
 * LASTQ items of those rows (chunks of [0, i]) and the LSE merge
 * (P:L641-642); no streaming pass.
 *   p->q, k, v: as for the other calls ([heads][N][d]).
 *   p->o:   Hq heads x r ROWS: O row t holds query token N - r + t.
 *   p->lse: optional [Hq][r] fp32, same row convention.
 * ws: >= ta_last_rows_workspace_size(p, last_q) bytes, 256-B aligned. */
size_t ta_last_rows_workspace_size(const ta_problem *p, int32_t last_q);
ta_status last_rows_attn_prefill(const ta_problem *p, int32_t last_q, void *ws, size_t ws_bytes,
                                 cudaStream_t stream);

/* ---- introspection (host only; no GPU needed) ---------------------------- */

/* Kept (i, j) pairs per head of the mask (tri == NULL -> dense causal).
 * TA_ERR_EMPTY_SEQUENCE / TA_ERR_PARAMS as above. */
ta_status ta_pair_count(int64_t seq_len, const ta_triangle *tri, int64_t *out_pairs_per_head);

/* Serialise the static block schedule the kernel would run
 * for (p, tri) on num_ctas persistent CTAs into host_buf.  Pointers inside *p
 * are not dereferenced (they may be NULL).  *inout_bytes: capacity in, bytes
 * needed/written out; host_buf == NULL or too small -> TA_ERR_WORKSPACE with
 * *inout_bytes set to the size needed. */
ta_status ta_schedule_export(const ta_problem *p, const ta_triangle *tri, int32_t num_ctas,
                             void *host_buf, size_t *inout_bytes);
/* Same for the final-layer last-rows mode (header kind field 2). */
ta_status ta_last_rows_schedule_export(const ta_problem *p, int32_t last_q, int32_t num_ctas,
                                       void *host_buf, size_t *inout_bytes);

const char *ta_status_str(ta_status s);
/* Detail of this thread's last non-OK return ("" if none). */
const char *ta_last_error(void);
int32_t ta_abi_version(void);
/* Free library-owned schedule/descriptor caches (device and host). */
void ta_release_caches(void);

/* Launch the LSE merge kernel with programmatic dependent launch after the
 * attention kernel (default on): the merge grid's launch overlaps the attention grid's
 * tail and its griddepcontrol.wait orders every read after the attention grid completes.
 * on = 0 launches it as a plain stream-ordered kernel.  Returns the previous setting. */
int32_t ta_set_pdl(int32_t on);

/* ---- kernel timing (used by bench.py) ------------------------------------ */
/* While enabled, every prefill call records CUDA events on its stream around the
 * attention kernel and around the merge kernel (library-owned events; the calls
 * stay asynchronous).  ta_profile_end() synchronises those events, writes the
 * summed device milliseconds and launch counts since ta_profile_begin(), and
 * disables recording.  Any out-pointer may be NULL. */
ta_status ta_profile_begin(void);
ta_status ta_profile_end(double *attn_ms, int64_t *attn_launches, double *merge_ms,
                         int64_t *merge_launches);

#ifdef __cplusplus
}
#endif
#endif /* TRIATTN_H_ */
