// schedule.h -- static block schedule of TriangleMix prefill attention (host side).
//
// Algorithm 1 (App. A.2) launches a static grid of
// ceil((N-N_last)/B_M) + S*ceil(N_last/B_M) programs per head: streaming
// programs for the upper rows and S split-K programs per last-row tile.  Here
// the same static work is enumerated once on the host as 16-byte ITEMS, costed
// in key columns and assigned to persistent CTAs by deterministic LPT
// (DESIGN.md section 4 is the normative spec; oracle/schedule_ref.py is an
// independent re-implementation of it used by the tests).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace ta {

enum ItemKind : uint8_t { kStream = 0, kLastQ = 1, kDense = 2 };

// One unit of work: NQT consecutive packed Q tiles ("a pair") of one kv head and
// a key range.  STREAM: [key_begin,key_end) is the sliding-window band, the sink
// [0, min(si, r1+1)) is implicit.  LASTQ: one split-K piece of [0, r1+1); `pad` is its
// chunk index (ordinal within the pair's span, < 256).  DENSE: [0, r1+1).
struct Item {
  uint8_t kind;
  uint8_t pad;  // LASTQ: chunk index; else 0
  uint16_t kv_head;
  uint32_t pair;
  uint32_t key_begin;
  uint32_t key_end;
};
static_assert(sizeof(Item) == 16, "item is 16 bytes");

constexpr int kTileRows = 128;      // tcgen05 M: packed rows per Q tile
constexpr int kTilesPerItem = 2;    // Q tiles sharing one K/V stream (two softmax warpgroups)
constexpr int kBlockKeys = 128;     // max keys per K/V block (tcgen05 N of QK^T)
constexpr int kKeyGranule = 16;     // MMA N granularity for M=128
constexpr int kSinkRows = 16;       // sink keys folded into a STREAM item's first block
// LPT cost of an item beyond its key columns (epilogue, pipeline turn-around; measured:
// a 5-block STREAM item costs about 190 columns more than its blocks inside a long item)
#ifndef TA_ITEM_OVERHEAD  // (overridable for schedule-policy experiments only; the oracle's
#define TA_ITEM_OVERHEAD 192  // schedule_ref.py mirrors the defaults)
#endif
constexpr int kItemOverhead = TA_ITEM_OVERHEAD;
constexpr uint32_t kScheduleMagic = 0x43534154u;  // "TASC"
constexpr uint32_t kScheduleVersion = 5;          // v2: water-filled LASTQ pieces; v4: + shared tail;
                                                  // v5: lock-step pieces of a head's last pairs
constexpr int kLockStepMax = 8;                   // lock-step groups for 2..8 last pairs per kv head
constexpr int kMaxCtas = 255;                     // chunk indices are u8 (<= 1 piece per CTA and span)
#ifndef TA_TAIL_PER_CTA  // (overridable for schedule-policy experiments only; schedule_ref.py mirrors 8)
#define TA_TAIL_PER_CTA 8
#endif
constexpr int kTailPerCta = TA_TAIL_PER_CTA;      // items per CTA moved to the shared tail (at most)
#ifndef TA_TAIL_DIV  // ... and at most (n + 1) / TA_TAIL_DIV of a CTA's n LPT items
#define TA_TAIL_DIV 3
#endif
constexpr int kTailDiv = TA_TAIL_DIV;
constexpr size_t kQueueBytes = 256;               // work-queue counter block at the workspace end

struct Geometry {
  int64_t n = 0;
  int hq = 0, hkv = 0, d = 0;
  int group = 0;        // G = Hq / Hkv
  int tile_tokens = 0;  // T = floor(128 / G) tokens per packed Q tile
  int pair_tokens = 0;  // P = kTilesPerItem * T tokens per item
  bool dense = false;
  bool last_only = false;  // final-layer mode: only the last `last` rows, all causal keys
  int si = 0, sl = 1, last = 1;
  int64_t num_pairs = 0;     // ceil(N / P)
  int64_t p_last0 = 0;       // first pair containing a row >= N - last (num_pairs if none)
  int64_t n_last_pairs = 0;  // num_pairs - p_last0 (triangle), 0 for dense
  int chunk_keys = 0;        // 0: LASTQ pieces have variable length (schedule v2)
  int s_max = 0;             // max pieces per last pair (set by build_schedule)
};

struct Schedule {
  Geometry g;
  int num_ctas = 0;
  std::vector<uint32_t> offsets;  // num_ctas + 1: CTA c's own list is items[offsets[c], offsets[c+1])
  std::vector<Item> items;        // the per-CTA lists (execution order), then the shared tail
  int64_t n_tail = 0;             // tail items items[offsets[num_ctas] ...], fetched dynamically
  std::vector<uint8_t> span_pieces;  // LASTQ pieces per (kvh, last pair), [hkv][n_last_pairs]
};

// Fills the geometry fields that do not depend on num_ctas. Returns false on bad input.
// s_max is set by build_schedule() (it depends on num_ctas and the LPT loads).
// last_only: final-layer mode, only LASTQ items over the last `last` rows (si, sl unused).
bool make_geometry(int64_t n, int hq, int hkv, int d, bool dense, int si, int sl, int last,
                   Geometry *g, std::string *err, bool last_only = false);
// Row range [r0, r1] (tokens) of pair p, clipped to N.
void pair_rows(const Geometry &g, int64_t p, int64_t *r0, int64_t *r1);
// Sum of 16-rounded block widths over the item's key blocks + kItemOverhead.
int64_t item_cost(const Geometry &g, const Item &it);
// Enumerate + LPT of STREAM/DENSE items + water-filling of the LASTQ work (DESIGN.md
// section 4).  1 <= num_ctas <= kMaxCtas.
Schedule build_schedule(const Geometry &g, int num_ctas);
std::vector<uint8_t> serialize(const Schedule &s);
// Partial-output slots (split-K workspace) and their byte size (g from build_schedule).
int64_t num_partial_slots(const Geometry &g);
size_t partial_bytes(const Geometry &g);
size_t workspace_bytes(const Geometry &g);

}  // namespace ta
