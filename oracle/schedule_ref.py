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
    LASTQ(kvh, p, c): [c*ck, min((c+1)*ck, r1+1)) for c < ceil((r1+1)/ck).
  dense: DENSE(kvh, p) = [0, r1+1).
  blocks: each key range cut at 128, width rounded up to 16; STREAM sink range first.
  cost = sum of block widths + 192 (per-item overhead: epilogue, pipeline turn-around).
  ck = largest power of two <= C_tot // (8 num_ctas) clamped to [512, 16384]
       (4 num_ctas in the last-rows mode)
       (C_tot: all STREAM items + one unsplit LASTQ item per last pair, all kv heads).
  canonical order: LASTQ (kvh, p, c) then STREAM/DENSE (kvh, p);
  LPT: stable sort by cost descending; each to least-loaded CTA, ties lowest id.
  bytes: 16 x u32 header, u32 offsets[num_ctas+1], 16-byte items
         {u8 kind, u8 0, u16 kvh, u32 pair, u32 key_begin, u32 key_end}.
"""
from __future__ import annotations

import struct

STREAM, LASTQ, DENSE = 0, 1, 2
MAGIC, VERSION = 0x43534154, 1



ITEM_OVERHEAD = 192  # LPT cost of an item beyond its key columns
CK_DIV = 8           # chunk_keys target: C_tot / (CK_DIV * num_ctas)
CK_DIV_LAST_ROWS = 4  # ... in the final-layer last-rows mode (LASTQ items only)

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
    kind, kvh, p, kb, ke = it
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


def chunk_keys(geo, num_ctas):
    if geo["dense"]:
        return 0
    tot = 0
    for p in range(0 if geo["last_rows"] else geo["p_last0"]):
        tot += cost(geo, stream_item(geo, 0, p))
    for p in range(geo["p_last0"], geo["pairs"]):
        tot += cost(geo, (LASTQ, 0, p, 0, rows(geo, p)[1] + 1))
    tot *= geo["hkv"]
    target = tot // ((CK_DIV_LAST_ROWS if geo["last_rows"] else CK_DIV) * num_ctas)
    ck = 512
    while ck * 2 <= target and ck * 2 <= 16384:
        ck *= 2
    return ck


def enumerate_items(geo, ck):
    items = []
    if geo["dense"]:
        for kvh in range(geo["hkv"]):
            for p in range(geo["pairs"]):
                items.append((DENSE, kvh, p, 0, rows(geo, p)[1] + 1))
        return items
    for kvh in range(geo["hkv"]):
        for p in range(geo["p_last0"], geo["pairs"]):
            span = rows(geo, p)[1] + 1
            for c in range(-(-span // ck)):
                items.append((LASTQ, kvh, p, c * ck, min((c + 1) * ck, span)))
    if not geo["last_rows"]:
        for kvh in range(geo["hkv"]):
            for p in range(geo["p_last0"]):
                items.append(stream_item(geo, kvh, p))
    return items


def schedule(n, hq, hkv, d, si, sl, last, dense, num_ctas, last_rows=False):
    """Returns (geo, ck, s_max, per_cta_lists)."""
    geo = geometry(n, hq, hkv, d, si, sl, last, dense, last_rows)
    ck = chunk_keys(geo, num_ctas)
    s_max = 0 if dense else -(-n // ck)
    items = enumerate_items(geo, ck)
    costs = [cost(geo, it) for it in items]
    order = sorted(range(len(items)), key=lambda i: (-costs[i], i))
    load = [0] * num_ctas
    per = [[] for _ in range(num_ctas)]
    for i in order:
        c = min(range(num_ctas), key=lambda x: (load[x], x))
        per[c].append(items[i])
        load[c] += costs[i]
    return geo, ck, s_max, per, load


def serialize(n, hq, hkv, d, si, sl, last, dense, num_ctas, last_rows=False) -> bytes:
    geo, ck, s_max, per, _ = schedule(n, hq, hkv, d, si, sl, last, dense, num_ctas, last_rows)
    nitems = sum(len(x) for x in per)
    kind = 1 if dense else (2 if geo["last_rows"] else 0)
    hdr = [MAGIC, VERSION, kind, n, hq, hkv, d, geo["si"], geo["sl"], geo["last"],
           geo["T"], 2, ck, num_ctas, nitems, s_max]
    out = struct.pack("<16I", *hdr)
    off = [0]
    for x in per:
        off.append(off[-1] + len(x))
    out += struct.pack("<%dI" % len(off), *off)
    for x in per:
        for kind, kvh, p, kb, ke in x:
            out += struct.pack("<BBHIII", kind, 0, kvh, p, kb, ke)
    return out


def parse(buf: bytes):
    """Decode the exported byte format into (header list, offsets, items)."""
    hdr = list(struct.unpack_from("<16I", buf, 0))
    num_ctas, nitems = hdr[13], hdr[14]
    off = list(struct.unpack_from("<%dI" % (num_ctas + 1), buf, 64))
    base = 64 + 4 * (num_ctas + 1)
    items = [struct.unpack_from("<BBHIII", buf, base + 16 * i) for i in range(nitems)]
    return hdr, off, [(k, kvh, p, kb, ke) for (k, _, kvh, p, kb, ke) in items]
