"""Static block schedule: byte identity with the independent enumerator, exact
coverage of the mask by brute force, LPT balance (SURVEY 8(c) 'Schedule' pin)."""
import random

import numpy as np
import pytest

import paper_2507_21526_b200 as ta
from oracle import masks, schedule_ref


CASES = [
    # n, hq, hkv, d, si, sl, last, dense, num_ctas
    (512, 1, 1, 64, 4, 64, 64, False, 148),
    (512, 1, 1, 64, 4, 64, 64, True, 148),
    (4096, 32, 8, 128, 8, 512, 128, False, 148),
    (4097, 28, 4, 128, 8, 512, 128, False, 148),
    (1000, 8, 2, 128, 0, 100, 1, False, 7),
    (129, 4, 4, 64, 16, 8, 200, False, 3),
    (7, 2, 1, 128, 8, 512, 128, False, 148),
    (1, 32, 8, 128, 8, 512, 128, False, 148),
    (32768, 32, 8, 128, 8, 512, 128, False, 148),
    (32768, 32, 8, 128, 8, 512, 128, True, 148),
    (32768, 4, 1, 128, 8, 512, 128, False, 148),   # one kv-head shard (8 GPUs)
    (1000, 32, 8, 128, 8, 512, 0, False, 148),     # StreamingMix: no last rows (reading R12)
    (4097, 28, 4, 128, 64, 128, 0, False, 148),    # StreamingMix, probe-style sink/window
    (777, 7, 7, 64, 64, 128, 64, False, 11),       # unfused 64-key sink
]


@pytest.mark.parametrize("case", CASES)
def test_export_bytes_equal_independent_enumerator(case):
    n, hq, hkv, d, si, sl, last, dense, nc = case
    got = ta.schedule_export(n, hq, hkv, d, nc, si, sl, last, dense)
    want = schedule_ref.serialize(n, hq, hkv, d, si, sl, last, dense, nc)
    assert got == want


def test_schedule_is_deterministic():
    a = ta.schedule_export(20000, 32, 8, 128, 148)
    b = ta.schedule_export(20000, 32, 8, 128, 148)
    assert a == b


def _block_keeps(geo, item, block, i):
    """Keys of one block that the kernel keeps for row i (DESIGN.md section 4.3 rule)."""
    kind, kvh, p, kb0, ke0 = item[:5]
    btype, kb, w = block
    si, sl, last, n = geo["si"], geo["sl"], geo["last"], geo["n"]
    keys = range(kb, kb + w)
    if kind == schedule_ref.STREAM:
        if btype == "fused":
            sink = [j for j in range(16) if j < si and j <= i]
            band = [j for j in range(kb, min(kb + w - 16, ke0)) if i - sl < j <= i]
            return sink + band
        if btype == "sink":
            return [j for j in keys if j < si and j <= i]
        return [j for j in keys if i - sl < j <= i and j < ke0]
    if kind == schedule_ref.DENSE:
        return [j for j in keys if j <= min(i, ke0 - 1)]
    # LASTQ: triangle predicate inside the chunk
    return [j for j in keys if kb0 <= j < ke0 and j <= i and (j < si or i - j < sl or i >= n - last)]


@pytest.mark.parametrize("seed", range(12))
def test_items_cover_mask_exactly_once(seed):
    rng = random.Random(seed)
    n = rng.randint(1, 1500)
    hkv = 1
    hq = rng.choice([1, 2, 4, 7, 8])
    si, sl, last = rng.randint(0, 40), rng.randint(1, 300), rng.randint(0, 300)
    dense = rng.random() < 0.25
    nc = rng.choice([1, 5, 148])
    geo, ck, s_max, per, _, tail = schedule_ref.schedule(n, hq, hkv, 64, si, sl, last, dense, nc)
    hits = np.zeros((n, n), dtype=np.int32)
    for lst in per + [tail]:
        for it in lst:
            r0, r1 = schedule_ref.rows(geo, it[2])
            for blk in schedule_ref.item_blocks(geo, it):
                assert blk[2] % 16 == 0 and 16 <= blk[2] <= 128, blk
                for i in range(r0, r1 + 1):
                    for j in _block_keeps(geo, it, blk, i):
                        hits[i, j] += 1
    want = masks.mask_vectorised(n, si, sl, last, dense)
    assert np.array_equal(hits, want.astype(np.int32))


@pytest.mark.parametrize("n,hq,hkv,bound", [
    (32768, 32, 8, 1.02), (131072, 32, 8, 1.01),          # 1 GPU
    (131072, 4, 1, 1.05), (65536, 4, 1, 1.05),            # Llama, one kv head (8-way shard)
    (131072, 3, 1, 1.05), (131072, 4, 1, 1.05),           # Qwen at 8 GPUs: 3 + 4 q-head split
    (65536, 3, 1, 1.05), (131072, 28, 4, 1.01),
    (32768, 8, 2, 1.05), (32768, 16, 4, 1.05),            # C2 at 4 / 2 GPUs
])
def test_lpt_balance_at_paper_configs(n, hq, hkv, bound):
    """Static lists + the shared tail fetched greedily (the kernel's end state), 148 CTAs."""
    geo, ck, s_max, per, load, tail = schedule_ref.schedule(n, hq, hkv, 128, 8, 512, 128, False, 148)
    fin = schedule_ref.final_loads(geo, load, tail)
    assert max(fin) / (sum(fin) / 148) <= bound, (n, hq, max(fin) / (sum(fin) / 148))


def test_shared_tail_absorbs_uneven_sm_speed():
    """Why the tail: with per-SM speeds spread +-2 % (measured on B200: CTAs with identical
    static lists differ by up to 3.7 % in cycles), fetching the tail dynamically keeps the
    finish times closer than running the same assignment statically."""
    geo, ck, s_max, per, load, tail = schedule_ref.schedule(131072, 32, 8, 128, 8, 512, 128, False, 148)
    assert len(tail) == 8 * 148
    rng = np.random.default_rng(0)
    speed = list(1.0 + rng.uniform(-0.02, 0.02, 148))
    dyn = schedule_ref.final_loads(geo, load, tail, speed)
    # the assignment the tail gets at equal speeds, frozen, then run at the uneven speeds
    import heapq
    heap = [(ld, c) for c, ld in enumerate(load)]
    heapq.heapify(heap)
    stat = list(load)
    for it in tail:
        t, c = heapq.heappop(heap)
        stat[c] += schedule_ref.cost(geo, it)
        heapq.heappush(heap, (t + schedule_ref.cost(geo, it), c))
    stat = [x / sp for x, sp in zip(stat, speed)]
    assert max(dyn) < max(stat)
    item = schedule_ref.cost(geo, tail[0])
    assert max(dyn) - min(dyn) <= 1.1 * item / min(speed)


def test_lpt_c2_eight_way_shard_at_stream_granularity():
    """C2 on an 8-way kv-head shard (N = 32768, 4 q heads): 510 equal STREAM items on 148
    CTAs force 66 CTAs to hold 4 of them; the Last Q-K work is water-filled into the
    others, whose pieces cost at least one 128-key block + the 192-column item overhead.
    The result is within one minimal piece of the 4-item floor (max / mean 1.06; the
    round-1 fixed-chunk LPT gave 1.14)."""
    geo, ck, s_max, per, load, tail = schedule_ref.schedule(32768, 4, 1, 128, 8, 512, 128, False, 148)
    fin = schedule_ref.final_loads(geo, load, tail)
    n_stream = sum(1 for lst in per + [tail] for it in lst if it[0] == schedule_ref.STREAM)
    stream_cost = schedule_ref.cost(geo, schedule_ref.stream_item(geo, 0, 10))
    floor = -(-n_stream // 148) * stream_cost
    assert max(fin) <= floor + 2 * schedule_ref.ITEM_OVERHEAD + 128 - 16
    assert max(fin) / (sum(fin) / 148) <= 1.07


@pytest.mark.parametrize("n,hq,hkv,nc", [(32768, 32, 8, 148), (32768, 4, 1, 148), (4097, 28, 4, 148),
                                         (1000, 8, 2, 7), (131072, 4, 1, 148)])
def test_lastq_pieces_tile_each_span_in_order(n, hq, hkv, nc):
    """Water-filled LASTQ pieces: per (kv head, last pair) they tile [0, r1+1) exactly, in key
    order, with chunk indices 0..k-1 (the merge's slots); s_max = the largest k."""
    geo, ck, s_max, per, load, tail = schedule_ref.schedule(n, hq, hkv, 128, 8, 512, 128, False, nc)
    assert all(it[0] != schedule_ref.LASTQ for it in tail)
    spans = {}
    for lst in per:
        for it in lst:
            if it[0] == schedule_ref.LASTQ:
                spans.setdefault((it[1], it[2]), []).append(it)
    assert s_max == max(len(v) for v in spans.values())
    for (kvh, p), its in spans.items():
        its.sort(key=lambda t: t[5])
        assert [t[5] for t in its] == list(range(len(its)))
        assert its[0][3] == 0 and its[-1][4] == schedule_ref.rows(geo, p)[1] + 1
        for a, b in zip(its, its[1:]):
            assert a[4] == b[3] and a[3] % 128 == 0


def test_last_rows_go_through_split_k():
    """Every row >= N-last belongs to a LASTQ pair (Algorithm 1 last-rows branch)."""
    geo, ck, s_max, per, _, tail = schedule_ref.schedule(32768, 32, 8, 128, 8, 512, 128, False, 148)
    last_pairs = {it[2] for lst in per for it in lst if it[0] == schedule_ref.LASTQ}
    for i in range(32768 - 128, 32768):
        assert i // geo["P"] in last_pairs
    hdr, off, items = schedule_ref.parse(ta.schedule_export(32768, 32, 8, 128, 148))
    assert hdr[0] == schedule_ref.MAGIC and hdr[1] == schedule_ref.VERSION == 5 and hdr[12] == len(tail) and hdr[15] == s_max
    assert off[-1] + len(tail) == len(items)


LAST_ROWS_CASES = [
    # n, hq, hkv, d, last, num_ctas
    (32768, 32, 8, 128, 128, 148),
    (131072, 32, 8, 128, 128, 148),
    (4097, 28, 4, 128, 100, 148),
    (300, 4, 1, 64, 1000, 7),   # last >= N: every row
    (1, 8, 8, 128, 128, 148),
]


@pytest.mark.parametrize("case", LAST_ROWS_CASES)
def test_last_rows_export_bytes_equal_independent_enumerator(case):
    """Final-layer mode: only LASTQ items of the last pairs, kind field 2."""
    n, hq, hkv, d, last, nc = case
    got = ta.last_rows_schedule_export(n, hq, hkv, d, nc, last)
    want = schedule_ref.serialize(n, hq, hkv, d, 8, 512, last, False, nc, last_rows=True)
    assert got == want
    hdr, off, items = schedule_ref.parse(got)
    assert hdr[2] == 2 and all(it[0] == schedule_ref.LASTQ for it in items)


@pytest.mark.parametrize("seed", range(6))
def test_last_rows_items_cover_last_rows_exactly_once(seed):
    """Every causal key of every row >= N - r is computed exactly once by the LASTQ chunks."""
    rng = random.Random(100 + seed)
    n = rng.randint(1, 1500)
    hq = rng.choice([1, 2, 4, 7, 8])
    last = rng.randint(1, 400)
    nc = rng.choice([1, 5, 148])
    geo, ck, s_max, per, _, tail = schedule_ref.schedule(n, hq, 1, 64, 8, 512, last, False, nc, last_rows=True)
    hits = np.zeros((n, n), dtype=np.int32)
    for lst in per + [tail]:
        for it in lst:
            assert it[0] == schedule_ref.LASTQ
            r0, r1 = schedule_ref.rows(geo, it[2])
            for blk in schedule_ref.item_blocks(geo, it):
                for i in range(max(r0, n - geo["last"]), r1 + 1):
                    for j in _block_keeps(geo, it, blk, i):
                        hits[i, j] += 1
    want = np.tril(np.ones((n, n), dtype=np.int32))
    want[: n - geo["last"]] = 0
    assert np.array_equal(hits, want)


def test_streamingmix_has_no_split_k():
    """last = 0: no LASTQ items and no workspace (StreamingMix deep layer)."""
    hdr, off, items = schedule_ref.parse(ta.schedule_export(4096, 32, 8, 128, 148, 8, 512, 0))
    assert items and all(it[0] == schedule_ref.STREAM for it in items)
    assert ta.workspace_size(4096, 32, 8, 128, 8, 512, 0) == 256   # the work-queue block only


@pytest.mark.parametrize("n,hq,hkv", [(131072, 32, 8), (32768, 4, 1), (131072, 28, 4), (65536, 3, 1)])
def test_lockstep_pieces_share_key_ranges(n, hq, hkv):
    """Schedule v5 (DESIGN 4.4 3'): a kv head's m last pairs are cut at the same key blocks,
    and the m pieces of each range sit on m different CTAs of one group (adjacent in the
    ascending-load order), so they run together and read each K/V block once from HBM."""
    geo, _, _, per, _, _ = schedule_ref.schedule(n, hq, hkv, 128, 8, 512, 128, False, 148)
    m = geo["pairs"] - geo["p_last0"]
    assert 2 <= m <= schedule_ref.LOCKSTEP_MAX
    where = {}
    for c, lst in enumerate(per):
        for it in lst:
            if it[0] == schedule_ref.LASTQ:
                where.setdefault((it[1], it[3] // 128), []).append((it[2], c))
    for (kvh, blk), lst in where.items():
        pairs = sorted(p for p, _ in lst)
        ctas = {c for _, c in lst}
        # every last pair whose span reaches this block has a piece starting here, each on its own CTA
        assert len(ctas) == len(lst) and len(set(pairs)) == len(pairs)
        assert len(lst) >= m - 1
