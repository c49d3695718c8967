// schedule.cpp -- enumeration, costing and LPT assignment of the static block
// schedule.  Pure host C++, no CUDA.
#include "schedule.h"

#include <algorithm>
#include <climits>
#include <cstring>
#include <numeric>
#include <queue>

namespace ta {

static inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

bool make_geometry(int64_t n, int hq, int hkv, int d, bool dense, int si, int sl, int last,
                   Geometry *g, std::string *err, bool last_only) {
  if (n < 1 || hq < 1 || hkv < 1 || hq % hkv != 0) {
    if (err) *err = "bad shape";
    return false;
  }
  Geometry r;
  r.n = n;
  r.hq = hq;
  r.hkv = hkv;
  r.d = d;
  r.group = hq / hkv;
  if (r.group > kTileRows) {
    if (err) *err = "Hq/Hkv > 128 cannot be packed into one 128-row tile";
    return false;
  }
  r.tile_tokens = kTileRows / r.group;
  r.pair_tokens = kTilesPerItem * r.tile_tokens;
  r.dense = dense;
  r.last_only = !dense && last_only;
  // Final-layer mode: the rows < N - last that share a pair with last rows are computed
  // with sink 0 / window 1 and never written.
  r.si = (dense || r.last_only) ? 0 : si;
  r.sl = (dense || r.last_only) ? 1 : sl;
  r.last = dense ? 1 : (r.last_only ? (int)std::min<int64_t>(last, n) : last);
  r.num_pairs = (n + r.pair_tokens - 1) / r.pair_tokens;
  if (dense) {
    r.p_last0 = r.num_pairs;
    r.n_last_pairs = 0;
  } else {
    // Rows >= N - last are "last rows" (reading R1); a pair holding any of them is
    // computed by the split-K pass over all of its causal keys (Algorithm 1).
    // last = 0 (StreamingMix, reading R12) has no last rows.
    r.p_last0 = r.last == 0 ? r.num_pairs : std::max<int64_t>(0, n - r.last) / r.pair_tokens;
    r.n_last_pairs = r.num_pairs - r.p_last0;
  }
  *g = r;
  return true;
}

void pair_rows(const Geometry &g, int64_t p, int64_t *r0, int64_t *r1) {
  *r0 = p * g.pair_tokens;
  *r1 = std::min<int64_t>((p + 1) * g.pair_tokens, g.n) - 1;
}

static int64_t range_cost(int64_t kb, int64_t ke) {
  int64_t c = 0;
  for (int64_t k = kb; k < ke; k += kBlockKeys)
    c += round_up(std::min<int64_t>(kBlockKeys, ke - k), kKeyGranule);
  return c;
}

int64_t item_cost(const Geometry &g, const Item &it) {
  int64_t c = kItemOverhead;
  if (it.kind == kStream) {
    int64_t r0, r1;
    pair_rows(g, it.pair, &r0, &r1);
    const int64_t s_end = std::min<int64_t>(g.si, r1 + 1);  // sink keys
    if (s_end > 0 && s_end <= kSinkRows) {
      // fused: block 0 = 16 sink columns + up to 112 band keys, then 128-key band blocks
      const int64_t first = kBlockKeys - kSinkRows;
      const int64_t len = (int64_t)it.key_end - it.key_begin;
      c += kSinkRows + round_up(std::min(first, len), kKeyGranule);
      if (len > first) c += range_cost(it.key_begin + first, it.key_end);
      return c;
    }
    c += range_cost(0, s_end);
  }
  c += range_cost(it.key_begin, it.key_end);
  return c;
}

static Item make_item(ItemKind kind, int kvh, int64_t pair, int64_t kb, int64_t ke) {
  Item it;
  it.kind = kind;
  it.pad = 0;
  it.kv_head = (uint16_t)kvh;
  it.pair = (uint32_t)pair;
  it.key_begin = (uint32_t)kb;
  it.key_end = (uint32_t)ke;
  return it;
}

static Item stream_item(const Geometry &g, int kvh, int64_t p) {
  int64_t r0, r1;
  pair_rows(g, p, &r0, &r1);
  // Sliding-window band relative to the tile (reading R5): keys [max(si, r0-sl+1), r1].
  int64_t b0 = std::max<int64_t>(g.si, r0 - g.sl + 1);
  int64_t b1 = r1 + 1;
  if (b0 > b1) b0 = b1;
  return make_item(kStream, kvh, p, b0, b1);
}

// Level of the Last Q-K water-filling: the smallest integer L such that the CTAs, each
// taking floor((L - load_c - kItemOverhead) / 128) blocks, hold all `nblocks` blocks.
static int64_t fill_level(const std::vector<int64_t> &load, int64_t nblocks) {
  auto cap = [&](int64_t L) {
    int64_t t = 0;
    for (int64_t x : load) t += std::max<int64_t>(0, (L - x - kItemOverhead) / kBlockKeys);
    return t;
  };
  int64_t lo = 0, hi = *std::max_element(load.begin(), load.end()) + kItemOverhead + kBlockKeys * nblocks;
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (cap(mid) >= nblocks)
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo;
}

Schedule build_schedule(const Geometry &g0, int num_ctas) {
  Schedule s;
  s.g = g0;
  Geometry &g = s.g;
  g.chunk_keys = 0;  // variable pieces (schedule version 2)
  g.s_max = 0;
  s.num_ctas = num_ctas;

  // 1. STREAM (triangle) or DENSE items, canonical order (kvh, pair), by LPT.
  std::vector<Item> canon;
  if (g.dense) {
    for (int kvh = 0; kvh < g.hkv; ++kvh)
      for (int64_t p = 0; p < g.num_pairs; ++p) {
        int64_t r0, r1;
        pair_rows(g, p, &r0, &r1);
        canon.push_back(make_item(kDense, kvh, p, 0, r1 + 1));
      }
  } else if (!g.last_only) {
    for (int kvh = 0; kvh < g.hkv; ++kvh)
      for (int64_t p = 0; p < g.p_last0; ++p) canon.push_back(stream_item(g, kvh, p));
  }
  const size_t ni = canon.size();
  std::vector<int64_t> cost(ni);
  for (size_t i = 0; i < ni; ++i) cost[i] = item_cost(g, canon[i]);
  std::vector<uint32_t> order(ni);
  std::iota(order.begin(), order.end(), 0u);
  std::stable_sort(order.begin(), order.end(),
                   [&](uint32_t a, uint32_t b) { return cost[a] > cost[b]; });
  // LPT: each item to the least-loaded CTA, ties to the lowest CTA id.
  typedef std::pair<int64_t, int> LoadCta;
  std::priority_queue<LoadCta, std::vector<LoadCta>, std::greater<LoadCta>> heap;
  for (int c = 0; c < num_ctas; ++c) heap.push(LoadCta(0, c));
  std::vector<std::vector<Item>> per(num_ctas);
  std::vector<int64_t> load(num_ctas, 0);
  for (uint32_t idx : order) {
    LoadCta top = heap.top();
    heap.pop();
    per[top.second].push_back(canon[idx]);
    load[top.second] = top.first + cost[idx];
    heap.push(LoadCta(load[top.second], top.second));
  }

  // 1b. Shared tail: the last min(kTailPerCta, (n + 1) / 3) items of each CTA's LPT list
  // (its smallest) leave the static assignment; the kernel's CTAs fetch them from a global
  // counter once their own lists are done, so per-SM speed differences (measured up to
  // 3.7 % between CTAs with identical lists) and cost-model error are absorbed at the end
  // (8 per CTA: -1.9 % max-over-CTA cycles at C3, -4.8 % at Qwen 128K vs no tail).
  std::vector<Item> tail;
  {
    std::vector<std::pair<int64_t, Item>> t;
    for (int c = 0; c < num_ctas; ++c) {
      const int k = std::min<int>(std::min<int>(kTailPerCta, ((int)per[c].size() + 1) / kTailDiv),
                                  (int)per[c].size());
      for (int i = 0; i < k; ++i) {
        const Item it = per[c].back();
        per[c].pop_back();
        const int64_t ic = item_cost(g, it);
        load[c] -= ic;
        t.push_back(std::make_pair(ic, it));
      }
    }
    // fetch order: cost descending, then (kind, kv head, pair)
    std::stable_sort(t.begin(), t.end(), [](const std::pair<int64_t, Item> &a, const std::pair<int64_t, Item> &b) {
      if (a.first != b.first) return a.first > b.first;
      if (a.second.kind != b.second.kind) return a.second.kind < b.second.kind;
      if (a.second.kv_head != b.second.kv_head) return a.second.kv_head < b.second.kv_head;
      return a.second.pair < b.second.pair;
    });
    for (auto &x : t) tail.push_back(x.second);
  }

  // 2. Water-filling of the Last Q-K work (Algorithm 1's split-K "last rows" programs,
  // P:L622-638; reading R7): the key spans [0, r1+1) of the last pairs, canonical order
  // (kvh, pair), in 128-key blocks, go to the CTAs in ascending (load, id) order, each up
  // to the common level; a take is cut at span ends into LASTQ pieces whose chunk index
  // (Item::pad) is their ordinal within the span.
  if (!g.dense && g.n_last_pairs > 0) {
    struct Span { int kvh; int64_t pair, keys, nblk; };
    std::vector<Span> spans;
    int64_t total = 0;
    for (int kvh = 0; kvh < g.hkv; ++kvh)
      for (int64_t p = g.p_last0; p < g.num_pairs; ++p) {
        int64_t r0, r1;
        pair_rows(g, p, &r0, &r1);
        const int64_t nb = (r1 + 1 + kBlockKeys - 1) / kBlockKeys;
        spans.push_back(Span{kvh, p, r1 + 1, nb});
        total += nb;
      }
    std::vector<int> cta(num_ctas);
    std::iota(cta.begin(), cta.end(), 0);
    std::stable_sort(cta.begin(), cta.end(), [&](int a, int b) { return load[a] < load[b]; });
    std::vector<int> pieces(spans.size(), 0);
    // Lock-step pieces (schedule version 5): with m = n_last_pairs in [2, kLockStepMax],
    // groups of m consecutive CTAs (ascending load) take the same key-block range from each
    // of a kv head's m last pairs, so the m pieces that read the same K/V blocks run at the
    // same time and share them through L2 (C3: DRAM reads 2.66 -> 2.18 GB per launch, cycles
    // unchanged).  Otherwise the single-span water-filling below.
    const int m = (int)g.n_last_pairs;
    if (m >= 2 && m <= kLockStepMax && num_ctas >= m) {
      const int ngroups = num_ctas / m;
      std::vector<int64_t> maxnb(g.hkv, 0);
      int64_t columns = 0;
      for (int h = 0; h < g.hkv; ++h) {
        for (int j = 0; j < m; ++j) maxnb[h] = std::max(maxnb[h], spans[h * m + j].nblk);
        columns += maxnb[h];
      }
      auto gcap = [&](int64_t L, int gi) {
        int64_t t = INT64_MAX;
        for (int j = 0; j < m; ++j) t = std::min(t, std::max<int64_t>(0, (L - load[cta[gi * m + j]] - kItemOverhead) / kBlockKeys));
        return t;
      };
      int64_t lo = 0, hi = *std::max_element(load.begin(), load.end()) + kItemOverhead + kBlockKeys * columns;
      while (lo < hi) {
        const int64_t mid = lo + (hi - lo) / 2;
        int64_t c = 0;
        for (int gi = 0; gi < ngroups; ++gi) c += gcap(mid, gi);
        if (c >= columns) hi = mid; else lo = mid + 1;
      }
      const int64_t L = lo;
      int h = 0;
      int64_t kcol = 0;
      for (int gi = 0; gi < ngroups && h < g.hkv; ++gi) {
        int64_t tg = gcap(L, gi);
        while (tg > 0 && h < g.hkv) {
          const int64_t t = std::min(tg, maxnb[h] - kcol);
          for (int j = 0; j < m; ++j) {
            const size_t sidx = (size_t)h * m + j;
            const Span &sp = spans[sidx];
            const int64_t b0 = kcol, b1 = std::min(kcol + t, sp.nblk);
            if (b1 <= b0) continue;
            Item it = make_item(kLastQ, sp.kvh, sp.pair, b0 * kBlockKeys, std::min<int64_t>(b1 * kBlockKeys, sp.keys));
            it.pad = (uint8_t)pieces[sidx]++;
            const int c = cta[gi * m + j];
            per[c].push_back(it);
            load[c] += item_cost(g, it);
          }
          kcol += t;
          tg -= t;
          if (kcol == maxnb[h]) {
            ++h;
            kcol = 0;
          }
        }
      }
    } else {
      const int64_t L = fill_level(load, total);
      size_t si = 0;
      int64_t off = 0, rem = total;
      for (int c : cta) {
        if (rem == 0) break;
        int64_t take = std::min(rem, std::max<int64_t>(0, (L - load[c] - kItemOverhead) / kBlockKeys));
        while (take > 0) {
          const Span &sp = spans[si];
          const int64_t k = std::min(take, sp.nblk - off);
          Item it = make_item(kLastQ, sp.kvh, sp.pair, off * kBlockKeys,
                              std::min<int64_t>((off + k) * kBlockKeys, sp.keys));
          it.pad = (uint8_t)pieces[si]++;
          per[c].push_back(it);
          load[c] += item_cost(g, it);
          off += k;
          take -= k;
          rem -= k;
          if (off == sp.nblk) {
            ++si;
            off = 0;
          }
        }
      }
    }
    g.s_max = *std::max_element(pieces.begin(), pieces.end());
    s.span_pieces.assign(pieces.begin(), pieces.end());
  }
  s.offsets.assign(num_ctas + 1, 0);
  s.items.reserve(ni + (size_t)num_ctas);
  for (int c = 0; c < num_ctas; ++c) {
    s.offsets[c] = (uint32_t)s.items.size();
#ifdef TA_LASTQ_FIRST  // (experiment) a CTA's LASTQ pieces before its STREAM items
    std::stable_partition(per[c].begin(), per[c].end(), [](const Item &it) { return it.kind == kLastQ; });
#endif
    s.items.insert(s.items.end(), per[c].begin(), per[c].end());
  }
  s.offsets[num_ctas] = (uint32_t)s.items.size();
  s.n_tail = (int64_t)tail.size();
  s.items.insert(s.items.end(), tail.begin(), tail.end());
  return s;
}

std::vector<uint8_t> serialize(const Schedule &s) {
  const Geometry &g = s.g;
  uint32_t hdr[16] = {kScheduleMagic,
                      kScheduleVersion,
                      (uint32_t)(g.dense ? 1 : (g.last_only ? 2 : 0)),
                      (uint32_t)g.n,
                      (uint32_t)g.hq,
                      (uint32_t)g.hkv,
                      (uint32_t)g.d,
                      (uint32_t)g.si,
                      (uint32_t)g.sl,
                      (uint32_t)g.last,
                      (uint32_t)g.tile_tokens,
                      (uint32_t)kTilesPerItem,
                      (uint32_t)s.n_tail,
                      (uint32_t)s.num_ctas,
                      (uint32_t)s.items.size(),
                      (uint32_t)g.s_max};
  std::vector<uint8_t> out(sizeof(hdr) + s.offsets.size() * 4 + s.items.size() * sizeof(Item));
  uint8_t *w = out.data();
  std::memcpy(w, hdr, sizeof(hdr));
  w += sizeof(hdr);
  std::memcpy(w, s.offsets.data(), s.offsets.size() * 4);
  w += s.offsets.size() * 4;
  if (!s.items.empty()) std::memcpy(w, s.items.data(), s.items.size() * sizeof(Item));
  return out;
}

int64_t num_partial_slots(const Geometry &g) {
  return g.dense ? 0 : (int64_t)g.hkv * g.n_last_pairs * g.s_max;  // s_max from build_schedule
}

size_t partial_bytes(const Geometry &g) {
  const int64_t slots = num_partial_slots(g);
  if (slots == 0) return 0;
  const int64_t rows = (int64_t)kTilesPerItem * kTileRows;
  const size_t o_bytes = (size_t)slots * rows * g.d * sizeof(float);
  const size_t lse_bytes = (size_t)slots * rows * sizeof(float);
  return round_up((int64_t)o_bytes, 256) + round_up((int64_t)lse_bytes, 256);
}

size_t workspace_bytes(const Geometry &g) {
  // split-K partials + the 256-byte work-queue block (the shared tail's fetch counter)
  return partial_bytes(g) + kQueueBytes;
}

}  // namespace ta
