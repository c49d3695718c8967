"""Independent enumerator of the static block schedule.  TEST INFRASTRUCTURE.

Re-derives, from the normative text of DESIGN.md section 4 (not from the C++),
the exact bytes ``ta_schedule_export`` must produce, plus the per-item key
blocks, so tests can check (a) byte identity and (b) by brute force that the
items cover every kept (row, key) pair of the mask exactly once.

Spec summary:
  G = Hq/Hkv, T = 128 // G, P = 2T tokens per item ("pair"), pairs = ceil(N/P).
  triangle: p_last0 = max(0, N-last) // P (= pairs when last = 0: StreamingMix has no
    last rows); pairs p >= p_last0 are LAST pairs.
  last_rows (final-layer mode): si = 0, sl = 1, last = min(last, N); only the
    LASTQ items of the last pairs (no STREAM items); header kind field 2.
    STREAM(kvh, p), p < p_last0: band [max(si, r0-sl+1), r1+1) (empty -> [r1+1, r1+1));
       sink [0, min(si, r1+1)) implicit.
  dense: DENSE(kvh, p) = [0, r1+1).
  blocks: each key range cut at 128, width rounded up to 16; STREAM sink range first.
  cost = sum of block widths + 192 (per-item overhead: epilogue, pipeline turn-around).
  1. LPT of the STREAM / DENSE items (canonical order (kvh, p)): stable sort by cost
     descending; each to the least-loaded CTA, ties to the lowest CTA id.
  2. Water-filling of the Last Q-K work (schedule version 2): the spans [0, r1+1) of the
     last pairs, canonical order (kvh, p), are cut into 128-key blocks; B = total blocks.
     Level L = the smallest integer with sum_c max(0, (L - load_c - 192) // 128) >= B.
     CTAs in order (load, id) ascending each take the next min(rem, cap_c) blocks of the
     span sequence; a take is cut at span ends into LASTQ(kvh, p) pieces
     [b0*128, min(b1*128, r1+1)) appended to that CTA's list; a piece's chunk index (u8
     item field `pad`) is its ordinal within its span.  s_max = max pieces per span.
  2'. (schedule version 5) When each kv head has m last pairs, 2 <= m <= 8 and
     num_ctas >= m, step 2 is replaced by lock-step pieces: the CTAs in (load, id) order
     form num_ctas // m groups of m; per head, maxnb = the most blocks of its m spans;
     group capacity gcap_g(L) = min over its CTAs of max(0, (L - load_c - 192) // 128);
     L = the smallest integer with sum_g gcap_g(L) >= sum_h maxnb_h.  Groups in order take
     block columns [k, k + t) of the current head (t = min(remaining capacity, maxnb - k)):
     the group's j-th CTA gets LASTQ(kvh, pair j) [k*128, min((k+t)*128, r1+1)) when that
     span has blocks there; k wraps to the next head at maxnb (a group may continue there).
  1b. (between 1 and 2; schedule version 4) Shared tail: each CTA's last
     min(8, (n + 1) // 3) LPT items (n = its LPT item count) leave its list (loads reduced
     before step 2); sorted by (cost desc, kind, kvh, pair) they form the tail that the
     kernel's CTAs fetch from a global counter after their own lists.
  bytes: 16 x u32 header (version 5; field 12 = tail entries), u32
         offsets[num_ctas+1], 16-byte items {u8 kind, u8 chunk, u16 kvh, u32 pair,
         u32 key_begin, u32 key_end}.
"""
from __future__ import annotations

import struct

STREAM, LASTQ, DENSE = 0, 1, 2
MAGIC, VERSION = 0x43534154, 5



ITEM_OVERHEAD = 192  # LPT cost of an item beyond its key columns
TAIL_PER_CTA = 8     # at most this many items per CTA go to the shared, dynamically fetched tail
LOCKSTEP_MAX = 8     # lock-step Last Q-K pieces for 2..8 last pairs per kv head (version 5)

def _r16(x):
    return -(-x // 16) * 16


def blocks_of(kb, ke):
    out = []
    k = kb
    while k < ke:
        out.append((k, _r16(min(128, ke - k))))
        k += 128
    return out


def geometry(n, hq, hkv, d, si, sl, last, dense, last_rows=False):
    g = hq // hkv
    t = 128 // g
    p = 2 * t
    pairs = -(-n // p)
    last_rows = bool(last_rows) and not dense
    if dense:
        si, sl, last = 0, 1, 1
        p_last0 = pairs
    else:
        if last_rows:
            si, sl, last = 0, 1, min(last, n)
        p_last0 = pairs if last == 0 else max(0, n - last) // p
    return dict(n=n, hq=hq, hkv=hkv, d=d, si=si, sl=sl, last=last, dense=dense, last_rows=last_rows,
                G=g, T=t, P=p, pairs=pairs, p_last0=p_last0)


def rows(geo, p):
    r0 = p * geo["P"]
    return r0, min(r0 + geo["P"], geo["n"]) - 1


def item_blocks(geo, it):
    """Key blocks of an item: (type, first key, width in S columns).

    type "fused": 16 sink columns (keys 0..15) followed by band keys from `first key`,
    width = 16 + round16(min(112, band length)); used for STREAM items whose sink span
    min(si, r1+1) is in 1..16.
    """
    kind, kvh, p, kb, ke = it[:5]
    bl = []
    if kind == STREAM:
        r0, r1 = rows(geo, p)
        s_end = min(geo["si"], r1 + 1)
        if 0 < s_end <= 16:
            n0 = min(112, ke - kb)
            bl.append(("fused", kb, 16 + _r16(n0)))
            return bl + [("main",) + b for b in blocks_of(kb + 112, ke)]
        bl += [("sink",) + b for b in blocks_of(0, s_end)]
    bl += [("main",) + b for b in blocks_of(kb, ke)]
    return bl


def cost(geo, it):
    return sum(b[2] for b in item_blocks(geo, it)) + ITEM_OVERHEAD


def stream_item(geo, kvh, p):
    r0, r1 = rows(geo, p)
    b0 = max(geo["si"], r0 - geo["sl"] + 1)
    b1 = r1 + 1
    return (STREAM, kvh, p, min(b0, b1), b1)


def base_items(geo):
    """STREAM (triangle) or DENSE items in canonical order (kvh, p); 6-tuples with pad 0."""
    items = []
    if geo["dense"]:
        for kvh in range(geo["hkv"]):
            for p in range(geo["pairs"]):
                items.append((DENSE, kvh, p, 0, rows(geo, p)[1] + 1, 0))
    elif not geo["last_rows"]:
        for kvh in range(geo["hkv"]):
            for p in range(geo["p_last0"]):
                items.append(stream_item(geo, kvh, p) + (0,))
    return items


def last_spans(geo):
    """(kvh, pair, keys) of every last pair, canonical order; keys = r1 + 1."""
    if geo["dense"]:
        return []
    return [(kvh, p, rows(geo, p)[1] + 1) for kvh in range(geo["hkv"])
            for p in range(geo["p_last0"], geo["pairs"])]


def fill_level(load, nblocks):
    """Smallest integer L with sum_c max(0, (L - load_c - ITEM_OVERHEAD) // 128) >= nblocks."""
    def cap(L):
        return sum(max(0, (L - x - ITEM_OVERHEAD) // 128) for x in load)
    lo, hi = 0, max(load) + ITEM_OVERHEAD + 128 * nblocks
    while lo < hi:
        mid = (lo + hi) // 2
        if cap(mid) >= nblocks:
            hi = mid
        else:
            lo = mid + 1
    return lo


def schedule(n, hq, hkv, d, si, sl, last, dense, num_ctas, last_rows=False):
    """Returns (geo, 0, s_max, per_cta_lists, loads, tail); items are 6-tuples
    (kind, kvh, pair, key_begin, key_end, chunk); loads are the static lists' costs."""
    geo = geometry(n, hq, hkv, d, si, sl, last, dense, last_rows)
    items = base_items(geo)
    costs = [cost(geo, it) for it in items]
    order = sorted(range(len(items)), key=lambda i: (-costs[i], i))
    load = [0] * num_ctas
    per = [[] for _ in range(num_ctas)]
    for i in order:
        c = min(range(num_ctas), key=lambda x: (load[x], x))
        per[c].append(items[i])
        load[c] += costs[i]
    tail = []
    for c in range(num_ctas):
        for _ in range(min(TAIL_PER_CTA, (len(per[c]) + 1) // 3)):
            it = per[c].pop()
            load[c] -= cost(geo, it)
            tail.append(it)
    tail.sort(key=lambda it: (-cost(geo, it), it[0], it[1], it[2]))
    spans = last_spans(geo)
    nblk = [-(-keys // 128) for (_, _, keys) in spans]
    total = sum(nblk)
    s_max = 0
    m = len(spans) // geo["hkv"] if spans else 0  # last pairs per kv head
    if total and 2 <= m <= LOCKSTEP_MAX and num_ctas >= m:
        # 2'. lock-step pieces (schedule version 5): groups of m consecutive CTAs in (load, id)
        # order take the same key-block range [k, k + t) from each of a head's m last pairs
        order = sorted(range(num_ctas), key=lambda x: (load[x], x))
        ngroups = num_ctas // m
        maxnb = [max(nblk[h * m + j] for j in range(m)) for h in range(geo["hkv"])]
        columns = sum(maxnb)

        def gcap(L, gi):
            return min(max(0, (L - load[order[gi * m + j]] - ITEM_OVERHEAD) // 128) for j in range(m))
        lo, hi = 0, max(load) + ITEM_OVERHEAD + 128 * columns
        while lo < hi:
            mid = (lo + hi) // 2
            if sum(gcap(mid, gi) for gi in range(ngroups)) >= columns:
                hi = mid
            else:
                lo = mid + 1
        L = lo
        pieces = [0] * len(spans)
        h, kcol = 0, 0
        for gi in range(ngroups):
            if h >= geo["hkv"]:
                break
            tg = gcap(L, gi)
            while tg > 0 and h < geo["hkv"]:
                t = min(tg, maxnb[h] - kcol)
                for j in range(m):
                    sidx = h * m + j
                    kvh, p, keys = spans[sidx]
                    b0, b1 = kcol, min(kcol + t, nblk[sidx])
                    if b1 <= b0:
                        continue
                    it = (LASTQ, kvh, p, b0 * 128, min(b1 * 128, keys), pieces[sidx])
                    c = order[gi * m + j]
                    per[c].append(it)
                    load[c] += cost(geo, it)
                    pieces[sidx] += 1
                kcol += t
                tg -= t
                if kcol == maxnb[h]:
                    h, kcol = h + 1, 0
        s_max = max(pieces)
    elif total:
        L = fill_level(load, total)
        caps = [max(0, (L - x - ITEM_OVERHEAD) // 128) for x in load]
        si_, off, rem = 0, 0, total
        pieces = [0] * len(spans)
        for c in sorted(range(num_ctas), key=lambda x: (load[x], x)):
            take = min(rem, caps[c])
            while take > 0:
                kvh, p, keys = spans[si_]
                k = min(take, nblk[si_] - off)
                it = (LASTQ, kvh, p, off * 128, min((off + k) * 128, keys), pieces[si_])
                per[c].append(it)
                load[c] += cost(geo, it)
                pieces[si_] += 1
                off += k
                take -= k
                rem -= k
                if off == nblk[si_]:
                    si_, off = si_ + 1, 0
            if rem == 0:
                break
        s_max = max(pieces)
    return geo, 0, s_max, per, load, tail


def final_loads(geo, load, tail, speed=None):
    """The kernel's end state: each CTA runs its own list, then fetches tail entries in
    order whenever it is free (greedy list scheduling; optional per-CTA speed factors)."""
    import heapq
    speed = speed or [1.0] * len(load)
    fin = [ld / sp for ld, sp in zip(load, speed)]
    heap = [(t, c) for c, t in enumerate(fin)]
    heapq.heapify(heap)
    for it in tail:
        t, c = heapq.heappop(heap)
        fin[c] = t + cost(geo, it) / speed[c]
        heapq.heappush(heap, (fin[c], c))
    return fin


def serialize(n, hq, hkv, d, si, sl, last, dense, num_ctas, last_rows=False) -> bytes:
    geo, ck, s_max, per, _, tail = schedule(n, hq, hkv, d, si, sl, last, dense, num_ctas, last_rows)
    nitems = sum(len(x) for x in per) + len(tail)
    kind = 1 if dense else (2 if geo["last_rows"] else 0)
    hdr = [MAGIC, VERSION, kind, n, hq, hkv, d, geo["si"], geo["sl"], geo["last"],
           geo["T"], 2, len(tail), num_ctas, nitems, s_max]
    out = struct.pack("<16I", *hdr)
    off = [0]
    for x in per:
        off.append(off[-1] + len(x))
    out += struct.pack("<%dI" % len(off), *off)
    for x in per + [tail]:
        for kind, kvh, p, kb, ke, ch in x:
            out += struct.pack("<BBHIII", kind, ch, kvh, p, kb, ke)
    return out


def parse(buf: bytes):
    """Decode the exported byte format into (header list, offsets, items): CTA c's list is
    items[off[c]:off[c+1]], the shared tail items[off[num_ctas]:] (hdr[12] entries)."""
    hdr = list(struct.unpack_from("<16I", buf, 0))
    num_ctas, nitems = hdr[13], hdr[14]
    off = list(struct.unpack_from("<%dI" % (num_ctas + 1), buf, 64))
    base = 64 + 4 * (num_ctas + 1)
    items = [struct.unpack_from("<BBHIII", buf, base + 16 * i) for i in range(nitems)]
    return hdr, off, [(k, kvh, p, kb, ke, ch) for (k, ch, kvh, p, kb, ke) in items]
