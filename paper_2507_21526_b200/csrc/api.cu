// api.cu -- the C ABI of include/triattn.h: validation, schedule/device caches,
// TMA descriptor encoding and kernel launch.  No torch types anywhere.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <atomic>
#include <chrono>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/triattn.h"
#include "kernel_params.h"
#include "schedule.h"

namespace {

// Launch ids for the in-kernel reset of the tail counter (kernel_params.h `epoch`).
uint32_t next_epoch() {
  static std::atomic<uint32_t> counter{0x9e3779b9u ^ (uint32_t)(uintptr_t)&counter ^
                                       (uint32_t)std::chrono::steady_clock::now().time_since_epoch().count()};
  uint32_t ep;
  do {
    ep = counter.fetch_add(1, std::memory_order_relaxed);
  } while (ep == 0u);
  return ep;
}


thread_local std::string g_last_error;

ta_status fail(ta_status s, const std::string &msg) {
  g_last_error = msg;
  return s;
}

// ------------------------------------------------------------------ validation
bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

ta_status validate_triangle(const ta_triangle *t) {
  if (!t) return fail(TA_ERR_NULL_ARG, "triangle parameters are NULL");
  if (t->sink < 0) return fail(TA_ERR_PARAMS, "sink < 0 (S:L39)");
  if (t->window < 1) return fail(TA_ERR_PARAMS, "window < 1 (S:L39)");
  if (t->last_q < 0) return fail(TA_ERR_PARAMS, "last_q < 0 (0 = StreamingMix, reading R12)");
  return TA_OK;
}

ta_status validate_shape(const ta_problem *p) {
  if (!p) return fail(TA_ERR_NULL_ARG, "problem is NULL");
  if (p->seq_len == 0) return fail(TA_ERR_EMPTY_SEQUENCE, "seq_len == 0 (S:L56)");
  if (p->seq_len < 0) return fail(TA_ERR_SHAPE, "seq_len < 0");
  if (p->num_q_heads < 1 || p->num_kv_heads < 1)
    return fail(TA_ERR_SHAPE, "head counts must be >= 1");
  if (p->num_q_heads % p->num_kv_heads != 0)
    return fail(TA_ERR_SHAPE, "num_q_heads % num_kv_heads != 0");
  if (p->head_dim != 64 && p->head_dim != 128)
    return fail(TA_ERR_UNSUPPORTED, "head_dim must be 64 or 128");
  if (p->num_q_heads / p->num_kv_heads > ta::kTileRows)
    return fail(TA_ERR_UNSUPPORTED, "Hq/Hkv > 128");
  if (p->seq_len >= (int64_t(1) << 31)) return fail(TA_ERR_UNSUPPORTED, "seq_len >= 2^31");
  if (p->num_kv_heads > 65535) return fail(TA_ERR_UNSUPPORTED, "num_kv_heads > 65535");
  return TA_OK;
}

ta_status validate_tensor(const char *name, const void *data, int64_t sh, int64_t st, int heads,
                          int64_t n, int d) {
  if (!data) return fail(TA_ERR_NULL_ARG, std::string(name) + ".data is NULL");
  if (st < d || (heads > 1 && sh < 1) || sh < 0)
    return fail(TA_ERR_SHAPE, std::string(name) + ": stride too small");
  if (heads > 1 && n > 1) {
    // views must not overlap: either head-major or token-major packing
    bool head_major = sh >= n * st;
    bool token_major = st >= (int64_t)heads * sh && sh >= d;
    if (!head_major && !token_major)
      return fail(TA_ERR_SHAPE, std::string(name) + ": overlapping head/token strides");
  }
  if (!aligned16(data)) return fail(TA_ERR_UNSUPPORTED, std::string(name) + ": not 16-byte aligned");
  if ((st * 2) % 16 != 0 || (sh * 2) % 16 != 0)
    return fail(TA_ERR_UNSUPPORTED, std::string(name) + ": stride*2 not a multiple of 16");
  return TA_OK;
}

// o_rows: token rows of the O view (N, or the last_q rows of the final-layer mode)
ta_status validate_problem(const ta_problem *p, int64_t o_rows = -1) {
  ta_status s = validate_shape(p);
  if (s != TA_OK) return s;
  const int64_t n = p->seq_len;
  const int d = p->head_dim;
  if (o_rows < 0) o_rows = n;
  if ((s = validate_tensor("q", p->q.data, p->q.stride_head, p->q.stride_token, p->num_q_heads, n, d)))
    return s;
  if ((s = validate_tensor("k", p->k.data, p->k.stride_head, p->k.stride_token, p->num_kv_heads, n, d)))
    return s;
  if ((s = validate_tensor("v", p->v.data, p->v.stride_head, p->v.stride_token, p->num_kv_heads, n, d)))
    return s;
  if ((s = validate_tensor("o", p->o.data, p->o.stride_head, p->o.stride_token, p->num_q_heads, o_rows, d)))
    return s;
  return TA_OK;
}

// ------------------------------------------------------------------ caches
struct DevSchedule {
  ta::Geometry g;
  ta::Item *d_items = nullptr;
  uint32_t *d_offsets = nullptr;
  uint8_t *d_span = nullptr;  // LASTQ pieces per (kvh, last pair), read by the merge
  int num_ctas = 0;
  int tail0 = 0, n_tail = 0;  // shared tail of the item list
};

typedef std::tuple<int, int64_t, int, int, int, int, int, int, int, int, int> SchedKey;
std::mutex g_mu;
std::map<SchedKey, DevSchedule> g_sched;
std::map<SchedKey, int> g_host_smax;  // s_max of host-built schedules (workspace queries)

SchedKey sched_key(int dev, const ta::Geometry &g, int num_ctas) {
  return SchedKey(dev, g.n, g.hq, g.hkv, g.d, g.dense ? 1 : 0, g.last_only ? 1 : 0, g.si, g.sl,
                  g.last, num_ctas);
}

// Persistent CTAs per launch: one per SM (chunk indices are u8: at most kMaxCtas).
int ctas_for(int sms) { return std::max(1, std::min(sms, ta::kMaxCtas)); }

// Geometry with s_max filled in (the water-filled schedule decides it), host only, cached.
ta::Geometry planned_geometry(const ta::Geometry &g0, int num_ctas) {
  ta::Geometry g = g0;
  if (g.dense) return g;
  const SchedKey key = sched_key(-1, g0, num_ctas);
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_host_smax.find(key);
    if (it != g_host_smax.end()) {
      g.s_max = it->second;
      return g;
    }
  }
  g = ta::build_schedule(g0, num_ctas).g;
  std::lock_guard<std::mutex> lk(g_mu);
  g_host_smax[key] = g.s_max;
  return g;
}

struct DeviceInfo {
  int sms = 0, major = 0, minor = 0;
};
std::map<int, DeviceInfo> g_dev;

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn g_encode = nullptr;

ta_status device_info(int *dev, DeviceInfo *info) {
  cudaError_t e = cudaGetDevice(dev);
  if (e != cudaSuccess) return fail(TA_ERR_CUDA, std::string("cudaGetDevice: ") + cudaGetErrorString(e));
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_dev.find(*dev);
  if (it == g_dev.end()) {
    DeviceInfo di;
    cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, *dev);
    cudaDeviceGetAttribute(&di.major, cudaDevAttrComputeCapabilityMajor, *dev);
    cudaDeviceGetAttribute(&di.minor, cudaDevAttrComputeCapabilityMinor, *dev);
    it = g_dev.emplace(*dev, di).first;
  }
  *info = it->second;
  if (info->major != 10 || info->minor != 0)
    return fail(TA_ERR_UNSUPPORTED, "device is not sm_100 (B200)");
  return TA_OK;
}

ta_status get_schedule(int dev, const ta::Geometry &g, int num_ctas, DevSchedule *out) {
  const SchedKey key = sched_key(dev, g, num_ctas);
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_sched.find(key);
  if (it != g_sched.end()) {
    *out = it->second;
    return TA_OK;
  }
  ta::Schedule s = ta::build_schedule(g, num_ctas);
  DevSchedule ds;
  ds.g = s.g;
  ds.num_ctas = num_ctas;
  ds.tail0 = (int)s.offsets[num_ctas];
  ds.n_tail = (int)s.n_tail;
  const size_t ib = std::max<size_t>(1, s.items.size()) * sizeof(ta::Item);
  const size_t ob = s.offsets.size() * sizeof(uint32_t);
  const size_t sb = std::max<size_t>(1, s.span_pieces.size());
  cudaError_t e = cudaMalloc(&ds.d_items, ib);
  if (e == cudaSuccess) e = cudaMalloc(&ds.d_offsets, ob);
  if (e == cudaSuccess) e = cudaMalloc(&ds.d_span, sb);
  if (e == cudaSuccess && !s.span_pieces.empty())
    e = cudaMemcpy(ds.d_span, s.span_pieces.data(), s.span_pieces.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !s.items.empty())
    e = cudaMemcpy(ds.d_items, s.items.data(), s.items.size() * sizeof(ta::Item), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(ds.d_offsets, s.offsets.data(), ob, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(ds.d_items);
    cudaFree(ds.d_offsets);
    cudaFree(ds.d_span);
    return fail(TA_ERR_CUDA, std::string("schedule upload: ") + cudaGetErrorString(e));
  }
  g_sched.emplace(key, ds);
  *out = ds;
  return TA_OK;
}

ta_status encode_map(CUtensorMap *m, const void *data, int64_t n, int heads, int d, int64_t sh,
                     int64_t st, uint32_t box_rows, uint32_t box_heads) {
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_encode) {
      void *fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
      if (e != cudaSuccess || !fn)
        return fail(TA_ERR_CUDA, "cuTensorMapEncodeTiled entry point not found");
      g_encode = reinterpret_cast<EncodeTiledFn>(fn);
    }
  }
  cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)n, (cuuint64_t)heads};
  cuuint64_t strides[2] = {(cuuint64_t)(st * 2), (cuuint64_t)(sh * 2)};
  if (heads == 1) strides[1] = (cuuint64_t)(st * 2) * (cuuint64_t)n;  // any legal value
  cuuint32_t box[3] = {64u, box_rows, box_heads};
  cuuint32_t estr[3] = {1u, 1u, 1u};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(data), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(TA_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return TA_OK;
}

#if defined(TA_TRACE) || defined(TA_CTA_CLOCK) || defined(TA_COUNT)
unsigned long long *g_trace_buf = nullptr;
size_t g_trace_bytes = sizeof(unsigned long long) * 65536 * 8;
#endif

std::atomic<int> g_pdl{1};  // merge launched with programmatic dependent launch

// ------------------------------------------------------------------ timing
struct Timing {
  bool on = false;
  std::vector<cudaEvent_t> pool;  // recycled events
  struct Rec { cudaEvent_t a0, a1, m1; };
  std::vector<Rec> recs;
};
Timing g_timing;

cudaEvent_t take_event() {
  if (!g_timing.pool.empty()) {
    cudaEvent_t e = g_timing.pool.back();
    g_timing.pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

enum Mode { kTriangle, kDenseMode, kLastRows };

// Geometry of a call: triangle (tri), dense, or the final-layer last-rows mode (last_q rows).
bool call_geometry(const ta_problem *p, const ta_triangle *tri, Mode mode, int32_t last_q,
                   ta::Geometry *g, std::string *err) {
  const bool dense = mode == kDenseMode;
  if (mode == kLastRows)
    return ta::make_geometry(p->seq_len, p->num_q_heads, p->num_kv_heads, p->head_dim, false, 0, 1,
                             last_q, g, err, true);
  return ta::make_geometry(p->seq_len, p->num_q_heads, p->num_kv_heads, p->head_dim, dense,
                           dense ? 0 : tri->sink, dense ? 1 : tri->window, dense ? 1 : tri->last_q, g,
                           err);
}

ta_status run(const ta_problem *p, const ta_triangle *tri, Mode mode, int32_t last_q, void *ws,
              size_t ws_bytes, cudaStream_t stream, const ta_out_tensor *extra_o = nullptr,
              int32_t n_extra = 0, const ta_out_tensor *mc_o = nullptr) {
  const bool dense = mode == kDenseMode;
  ta_status s = validate_shape(p);
  if (s != TA_OK) return s;
  if (mode == kLastRows && last_q < 1) return fail(TA_ERR_PARAMS, "last_q < 1 (final-layer rows)");
  const int64_t o_rows = mode == kLastRows ? std::min<int64_t>(last_q, p->seq_len) : p->seq_len;
  if ((s = validate_problem(p, o_rows)) != TA_OK) return s;
  if (mode == kTriangle && (s = validate_triangle(tri)) != TA_OK) return s;
  // f2: extra output destinations, validated like p->o before anything is enqueued
  if (n_extra < 0 || n_extra > ta::kMaxExtraOut || (n_extra > 0 && mode == kLastRows))
    return fail(TA_ERR_PARAMS, "n_extra must be in [0, " + std::to_string(ta::kMaxExtraOut) +
                                   "] (and 0 for the last-rows mode)");
  if (n_extra > 0 && !extra_o) return fail(TA_ERR_NULL_ARG, "extra_o is NULL");
  for (int e = 0; e < n_extra; ++e)
    if ((s = validate_tensor("extra_o", extra_o[e].data, extra_o[e].stride_head,
                             extra_o[e].stride_token, p->num_q_heads, o_rows, p->head_dim)))
      return s;
  if (mc_o && (s = validate_tensor("mc_o", mc_o->data, mc_o->stride_head, mc_o->stride_token,
                                   p->num_q_heads, o_rows, p->head_dim)))
    return s;
  int dev;
  DeviceInfo di;
  if ((s = device_info(&dev, &di)) != TA_OK) return s;
  ta::Geometry g;
  std::string err;
  if (!call_geometry(p, tri, mode, last_q, &g, &err)) return fail(TA_ERR_SHAPE, err);
  // The schedule (host build + one upload per device and signature, cached) fixes s_max
  // and so the workspace size; nothing is enqueued before the checks below.
  DevSchedule ds;
  if ((s = get_schedule(dev, g, ctas_for(di.sms), &ds)) != TA_OK) return s;
  const size_t need = ta::workspace_bytes(ds.g);
  if (need > 0) {
    if (!ws) return fail(TA_ERR_WORKSPACE, "workspace is NULL");
    if (ws_bytes < need) return fail(TA_ERR_WORKSPACE, "workspace too small: need " + std::to_string(need));
    if (reinterpret_cast<uintptr_t>(ws) & 255u) return fail(TA_ERR_WORKSPACE, "workspace not 256-byte aligned");
  }

  ta::AttnParams prm;
  std::memset(&prm, 0, sizeof(prm));
  const int G = g.group, T = g.tile_tokens;
  if ((s = encode_map(&prm.tm_q, p->q.data, g.n, g.hq, g.d, p->q.stride_head, p->q.stride_token, T, G)))
    return s;
  if ((s = encode_map(&prm.tm_o, p->o.data, o_rows, g.hq, g.d, p->o.stride_head, p->o.stride_token, T, G)))
    return s;
  if ((s = encode_map(&prm.tm_k, p->k.data, g.n, g.hkv, g.d, p->k.stride_head, p->k.stride_token,
                      ta::kBlockKeys, 1)))
    return s;
  if ((s = encode_map(&prm.tm_v, p->v.data, g.n, g.hkv, g.d, p->v.stride_head, p->v.stride_token,
                      ta::kBlockKeys, 1)))
    return s;
  if ((s = encode_map(&prm.tm_kb, p->k.data, g.n, g.hkv, g.d, p->k.stride_head, p->k.stride_token,
                      ta::kBlockKeys - ta::kSinkRows, 1)))
    return s;
  if ((s = encode_map(&prm.tm_vb, p->v.data, g.n, g.hkv, g.d, p->v.stride_head, p->v.stride_token,
                      ta::kBlockKeys - ta::kSinkRows, 1)))
    return s;
  if ((s = encode_map(&prm.tm_ks, p->k.data, g.n, g.hkv, g.d, p->k.stride_head, p->k.stride_token,
                      ta::kSinkRows, 1)))
    return s;
  if ((s = encode_map(&prm.tm_vs, p->v.data, g.n, g.hkv, g.d, p->v.stride_head, p->v.stride_token,
                      ta::kSinkRows, 1)))
    return s;
  prm.o = p->o.data;
  prm.o_sh = p->o.stride_head;
  prm.o_st = p->o.stride_token;
  prm.n_ox = n_extra;
  for (int e = 0; e < n_extra; ++e) {
    if ((s = encode_map(&prm.tm_ox[e], extra_o[e].data, o_rows, g.hq, g.d, extra_o[e].stride_head,
                        extra_o[e].stride_token, T, G)))
      return s;
    prm.ox[e] = extra_o[e].data;
    prm.ox_sh[e] = extra_o[e].stride_head;
    prm.ox_st[e] = extra_o[e].stride_token;
  }
  if (mc_o) {
    prm.mc_o = mc_o->data;
    prm.mc_sh = mc_o->stride_head;
    prm.mc_st = mc_o->stride_token;
  }
  prm.lse = p->lse;
  const size_t pbytes = ta::partial_bytes(ds.g);
  if (pbytes > 0) {
    const int64_t slots = ta::num_partial_slots(ds.g);
    const size_t o_bytes = ((size_t)slots * 2 * ta::kTileRows * g.d * 4 + 255) / 256 * 256;
    prm.part_o = reinterpret_cast<float *>(ws);
    prm.part_lse = reinterpret_cast<float *>(reinterpret_cast<uint8_t *>(ws) + o_bytes);
  }
  prm.queue = reinterpret_cast<uint32_t *>(reinterpret_cast<uint8_t *>(ws) + pbytes);
  prm.items = ds.d_items;
  prm.offsets = ds.d_offsets;
  prm.tail0 = ds.tail0;
  prm.n_tail = ds.n_tail;
  prm.n = (int)g.n;
  prm.hq = g.hq;
  prm.group = G;
  prm.tile_tokens = T;
  prm.pair_tokens = g.pair_tokens;
  prm.si = g.si;
  prm.sl = g.sl;
  prm.last = g.last;
  prm.dense = dense ? 1 : 0;
  prm.last_only = g.last_only ? 1 : 0;
  prm.o_row0 = (int)(g.n - o_rows);
  prm.p_last0 = (int)ds.g.p_last0;
  prm.n_last_pairs = (int)ds.g.n_last_pairs;
  prm.chunk_keys = ds.g.chunk_keys;
  prm.s_max = ds.g.s_max;
  prm.span_pieces = ds.d_span;
  const float scale = p->softmax_scale > 0.f ? p->softmax_scale : 1.0f / std::sqrt((float)g.d);
  prm.scale = scale;
  prm.scale_log2 = scale * 1.4426950408889634f;

  std::unique_lock<std::mutex> tlk(g_mu, std::defer_lock);
  Timing::Rec rec{nullptr, nullptr, nullptr};
  if (g_timing.on) {
    tlk.lock();
    rec.a0 = take_event();
    rec.a1 = take_event();
    cudaEventRecord(rec.a0, stream);
  }
#if defined(TA_CTA_CLOCK)
  {  // per-CTA elapsed SM cycles of this launch (kernel-variant comparisons independent of clocks)
    static unsigned long long *cbuf = nullptr;
    if (!cbuf) cudaMalloc(&cbuf, sizeof(unsigned long long) * 65536 * 8);
    prm.trace = cbuf;
    g_trace_buf = cbuf;
  }
#endif
#if defined(TA_COUNT)
  {  // per-(q head, token) counters {admitted pairs, computed S columns} (u32 pairs)
    static unsigned long long *kbuf = nullptr;
    static size_t kcap = 0;
    const size_t need = sizeof(uint32_t) * 2 * (size_t)g.hq * (size_t)g.n;
    if (need > kcap) {
      if (kbuf) cudaFree(kbuf);
      if (cudaMalloc(&kbuf, need) != cudaSuccess) return fail(TA_ERR_CUDA, "count buffer");
      kcap = need;
    }
    cudaMemsetAsync(kbuf, 0, need, stream);
    prm.trace = kbuf;
    g_trace_buf = kbuf;
    g_trace_bytes = need;
  }
#endif
#ifdef TA_TRACE
  {
    static unsigned long long *tbuf = nullptr;
    if (!tbuf) cudaMalloc(&tbuf, sizeof(unsigned long long) * 65536 * 8);
    cudaMemsetAsync(tbuf, 0, sizeof(unsigned long long) * 65536 * 8, stream);
    prm.trace = tbuf;
    const char *e = getenv("TA_TRACE_CTA");
    prm.trace_cta = e ? atoi(e) : 0;
    g_trace_buf = tbuf;
  }
#endif
  // The shared tail's fetch counter (in the caller's workspace, so calls on different
  // streams never share it) is reset by the kernel itself: CTA 0 swaps the 64-bit word to
  // {this launch's epoch, 0}, and a ticket is valid only if it carries that epoch
  // (kernel_params.h).  No memset is enqueued before the launch.  Epochs are
  // distinct for 2^32 launches per process and start at a per-process salt, so a fresh
  // workspace's leftover bytes do not look current.
  prm.epoch = next_epoch();
#ifdef TA_QUEUE_MEMSET  // (experiment) the round-2 memset reset, 32-bit tickets
  cudaMemsetAsync(prm.queue, 0, sizeof(uint32_t), stream);
#endif
  cudaError_t e = ta::launch_attention(prm, g.d, ds.num_ctas, stream);
  if (e != cudaSuccess) return fail(TA_ERR_CUDA, std::string("attention launch: ") + cudaGetErrorString(e));
  if (rec.a1) cudaEventRecord(rec.a1, stream);
  if (!dense && ds.g.n_last_pairs > 0) {
    e = ta::launch_merge(prm, g.d, g.hkv, stream, g_pdl.load(std::memory_order_relaxed) != 0);
    if (e != cudaSuccess) return fail(TA_ERR_CUDA, std::string("merge launch: ") + cudaGetErrorString(e));
    if (rec.a0) {
      rec.m1 = take_event();
      cudaEventRecord(rec.m1, stream);
    }
  }
  if (rec.a0) g_timing.recs.push_back(rec);
  return TA_OK;
}

size_t ws_size(const ta_problem *p, const ta_triangle *tri, Mode mode, int32_t last_q) {
  if (validate_shape(p) != TA_OK) return 0;
  if (mode == kTriangle && (!tri || validate_triangle(tri) != TA_OK)) return 0;
  if (mode == kLastRows && last_q < 1) return 0;
  ta::Geometry g;
  if (!call_geometry(p, tri, mode, last_q, &g, nullptr)) return 0;
  int sms = 148;  // B200; used when no device is visible (host-only callers)
  int dev;
  if (cudaGetDevice(&dev) == cudaSuccess) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0) sms = v;
  } else {
    cudaGetLastError();
  }
  return ta::workspace_bytes(planned_geometry(g, ctas_for(sms)));
}

}  // namespace

extern "C" {

size_t ta_workspace_size(const ta_problem *p, const ta_triangle *tri) {
  try {
    return ws_size(p, tri, tri ? kTriangle : kDenseMode, 0);
  } catch (...) {
    return 0;
  }
}

ta_status triangle_attn_prefill(const ta_problem *p, const ta_triangle *tri, void *ws,
                                size_t ws_bytes, cudaStream_t stream) {
  try {
    if (!tri) return fail(TA_ERR_NULL_ARG, "triangle parameters are NULL");
    return run(p, tri, kTriangle, 0, ws, ws_bytes, stream);
  } catch (const std::exception &ex) {
    return fail(TA_ERR_CUDA, ex.what());
  } catch (...) {
    return fail(TA_ERR_CUDA, "unknown exception");
  }
}

ta_status triangle_attn_prefill_multi(const ta_problem *p, const ta_triangle *tri,
                                      const ta_out_tensor *extra_o, int32_t n_extra, void *ws,
                                      size_t ws_bytes, cudaStream_t stream) {
  try {
    if (!tri) return fail(TA_ERR_NULL_ARG, "triangle parameters are NULL");
    return run(p, tri, kTriangle, 0, ws, ws_bytes, stream, extra_o, n_extra);
  } catch (const std::exception &ex) {
    return fail(TA_ERR_CUDA, ex.what());
  } catch (...) {
    return fail(TA_ERR_CUDA, "unknown exception");
  }
}

ta_status triangle_attn_prefill_multicast(const ta_problem *p, const ta_triangle *tri,
                                          const ta_out_tensor *mc_o, void *ws, size_t ws_bytes,
                                          cudaStream_t stream) {
  try {
    if (!tri) return fail(TA_ERR_NULL_ARG, "triangle parameters are NULL");
    if (!mc_o) return fail(TA_ERR_NULL_ARG, "mc_o is NULL");
    return run(p, tri, kTriangle, 0, ws, ws_bytes, stream, nullptr, 0, mc_o);
  } catch (const std::exception &ex) {
    return fail(TA_ERR_CUDA, ex.what());
  } catch (...) {
    return fail(TA_ERR_CUDA, "unknown exception");
  }
}

ta_status dense_attn_prefill_multicast(const ta_problem *p, const ta_out_tensor *mc_o, void *ws,
                                       size_t ws_bytes, cudaStream_t stream) {
  try {
    if (!mc_o) return fail(TA_ERR_NULL_ARG, "mc_o is NULL");
    return run(p, nullptr, kDenseMode, 0, ws, ws_bytes, stream, nullptr, 0, mc_o);
  } catch (const std::exception &ex) {
    return fail(TA_ERR_CUDA, ex.what());
  } catch (...) {
    return fail(TA_ERR_CUDA, "unknown exception");
  }
}

ta_status dense_attn_prefill_multi(const ta_problem *p, const ta_out_tensor *extra_o,
                                   int32_t n_extra, void *ws, size_t ws_bytes, cudaStream_t stream) {
  try {
    return run(p, nullptr, kDenseMode, 0, ws, ws_bytes, stream, extra_o, n_extra);
  } catch (const std::exception &ex) {
    return fail(TA_ERR_CUDA, ex.what());
  } catch (...) {
    return fail(TA_ERR_CUDA, "unknown exception");
  }
}

ta_status dense_attn_prefill(const ta_problem *p, void *ws, size_t ws_bytes, cudaStream_t stream) {
  try {
    return run(p, nullptr, kDenseMode, 0, ws, ws_bytes, stream);
  } catch (const std::exception &ex) {
    return fail(TA_ERR_CUDA, ex.what());
  } catch (...) {
    return fail(TA_ERR_CUDA, "unknown exception");
  }
}

ta_status ta_layer_attn_prefill(int32_t layer, int32_t tri_start, const ta_problem *p,
                                const ta_triangle *tri, void *ws, size_t ws_bytes,
                                cudaStream_t stream) {
  if (layer < 0) return fail(TA_ERR_PARAMS, "layer < 0");
  if (tri_start < 0) return fail(TA_ERR_PARAMS, "tri_start < 0 (S:L40)");
  // P:L255-269 with reading R2: layers [0, tri_start) dense, [tri_start, L) triangle.
  if (layer < tri_start) return dense_attn_prefill(p, ws, ws_bytes, stream);
  return triangle_attn_prefill(p, tri, ws, ws_bytes, stream);
}

ta_status ta_pair_count(int64_t seq_len, const ta_triangle *tri, int64_t *out) {
  if (!out) return fail(TA_ERR_NULL_ARG, "out_pairs_per_head is NULL");
  if (seq_len == 0) return fail(TA_ERR_EMPTY_SEQUENCE, "seq_len == 0 (S:L56)");
  if (seq_len < 0) return fail(TA_ERR_SHAPE, "seq_len < 0");
  const int64_t n = seq_len;
  if (!tri) {
    *out = n * (n + 1) / 2;
    return TA_OK;
  }
  ta_status s = validate_triangle(tri);
  if (s != TA_OK) return s;
  // Row by row over the section definitions: rows i < N-last keep the
  // streaming keys min(i+1, si+sl); rows i >= N-last keep all i+1 causal keys.
  const int64_t w = (int64_t)tri->sink + tri->window;
  const int64_t r = std::max<int64_t>(0, n - tri->last_q);
  int64_t stream_pairs = r <= w ? r * (r + 1) / 2 : w * (w + 1) / 2 + (r - w) * w;
  *out = stream_pairs + n * (n + 1) / 2 - r * (r + 1) / 2;
  return TA_OK;
}

namespace {
ta_status export_schedule(const ta_problem *p, const ta_triangle *tri, Mode mode, int32_t last_q,
                          int32_t num_ctas, void *host_buf, size_t *inout_bytes) {
  try {
    if (!inout_bytes) return fail(TA_ERR_NULL_ARG, "inout_bytes is NULL");
    ta_status s = validate_shape(p);
    if (s != TA_OK) return s;
    if (mode == kTriangle && (s = validate_triangle(tri)) != TA_OK) return s;
    if (mode == kLastRows && last_q < 1) return fail(TA_ERR_PARAMS, "last_q < 1 (final-layer rows)");
    if (num_ctas < 1 || num_ctas > ta::kMaxCtas)
      return fail(TA_ERR_PARAMS, "num_ctas must be in [1, " + std::to_string(ta::kMaxCtas) + "]");
    ta::Geometry g;
    std::string err;
    if (!call_geometry(p, tri, mode, last_q, &g, &err)) return fail(TA_ERR_SHAPE, err);
    std::vector<uint8_t> bytes = ta::serialize(ta::build_schedule(g, num_ctas));
    const size_t cap = *inout_bytes;
    *inout_bytes = bytes.size();
    if (!host_buf || cap < bytes.size()) return fail(TA_ERR_WORKSPACE, "buffer too small");
    std::memcpy(host_buf, bytes.data(), bytes.size());
    return TA_OK;
  } catch (...) {
    return fail(TA_ERR_CUDA, "exception in ta_schedule_export");
  }
}
}  // namespace

ta_status ta_schedule_export(const ta_problem *p, const ta_triangle *tri, int32_t num_ctas,
                             void *host_buf, size_t *inout_bytes) {
  return export_schedule(p, tri, tri ? kTriangle : kDenseMode, 0, num_ctas, host_buf, inout_bytes);
}

size_t ta_last_rows_workspace_size(const ta_problem *p, int32_t last_q) {
  try {
    return ws_size(p, nullptr, kLastRows, last_q);
  } catch (...) {
    return 0;
  }
}

ta_status last_rows_attn_prefill(const ta_problem *p, int32_t last_q, void *ws, size_t ws_bytes,
                                 cudaStream_t stream) {
  try {
    return run(p, nullptr, kLastRows, last_q, ws, ws_bytes, stream);
  } catch (const std::exception &ex) {
    return fail(TA_ERR_CUDA, ex.what());
  } catch (...) {
    return fail(TA_ERR_CUDA, "unknown exception");
  }
}

ta_status ta_last_rows_schedule_export(const ta_problem *p, int32_t last_q, int32_t num_ctas,
                                       void *host_buf, size_t *inout_bytes) {
  return export_schedule(p, nullptr, kLastRows, last_q, num_ctas, host_buf, inout_bytes);
}

const char *ta_status_str(ta_status s) {
  switch (s) {
    case TA_OK: return "TA_OK";
    case TA_ERR_NULL_ARG: return "TA_ERR_NULL_ARG";
    case TA_ERR_EMPTY_SEQUENCE: return "TA_ERR_EMPTY_SEQUENCE";
    case TA_ERR_SHAPE: return "TA_ERR_SHAPE";
    case TA_ERR_PARAMS: return "TA_ERR_PARAMS";
    case TA_ERR_UNSUPPORTED: return "TA_ERR_UNSUPPORTED";
    case TA_ERR_WORKSPACE: return "TA_ERR_WORKSPACE";
    case TA_ERR_CUDA: return "TA_ERR_CUDA";
  }
  return "TA_ERR_UNKNOWN";
}

const char *ta_last_error(void) { return g_last_error.c_str(); }

int32_t ta_abi_version(void) { return TA_ABI_VERSION; }

ta_status ta_profile_begin(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_timing.on = true;
  g_timing.recs.clear();
  return TA_OK;
}

ta_status ta_profile_end(double *attn_ms, int64_t *attn_launches, double *merge_ms,
                         int64_t *merge_launches) {
  std::lock_guard<std::mutex> lk(g_mu);
  double a = 0, m = 0;
  int64_t na = 0, nm = 0;
  ta_status st = TA_OK;
  for (auto &r : g_timing.recs) {
    float t = 0.f;
    if (cudaEventSynchronize(r.a1) != cudaSuccess || cudaEventSynchronize(r.a0) != cudaSuccess) {
      st = fail(TA_ERR_CUDA, "event synchronize failed");
    } else if (cudaEventElapsedTime(&t, r.a0, r.a1) == cudaSuccess) {
      a += t;
      ++na;
    }
    if (r.m1 && cudaEventSynchronize(r.m1) == cudaSuccess &&
        cudaEventElapsedTime(&t, r.a1, r.m1) == cudaSuccess) {
      m += t;
      ++nm;
    }
    g_timing.pool.push_back(r.a0);
    g_timing.pool.push_back(r.a1);
    if (r.m1) g_timing.pool.push_back(r.m1);
  }
  g_timing.recs.clear();
  g_timing.on = false;
  if (attn_ms) *attn_ms = a;
  if (attn_launches) *attn_launches = na;
  if (merge_ms) *merge_ms = m;
  if (merge_launches) *merge_launches = nm;
  return st;
}

#if defined(TA_TRACE) || defined(TA_CTA_CLOCK) || defined(TA_COUNT)
/* Debug builds only: copy the last launch's timeline (TA_TRACE), per-CTA cycle counts
   (TA_CTA_CLOCK) or per-row pair counters (TA_COUNT: u32 {admitted, computed} per
   [q head][token]) to the host.  Synchronises the device. */
ta_status ta_debug_trace_read(void *host, size_t cap) {
  if (!g_trace_buf) return TA_ERR_CUDA;
  const size_t n = g_trace_bytes;
  cudaMemcpy(host, g_trace_buf, cap < n ? cap : n, cudaMemcpyDeviceToHost);
  return TA_OK;
}
#endif

int32_t ta_set_pdl(int32_t on) {
  return g_pdl.exchange(on ? 1 : 0);
}

void ta_release_caches(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto &kv : g_sched) {
    cudaFree(kv.second.d_items);
    cudaFree(kv.second.d_offsets);
    cudaFree(kv.second.d_span);
  }
  g_sched.clear();
  g_host_smax.clear();
}

}  // extern "C"
