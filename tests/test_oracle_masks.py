"""Pins for oracle/masks.py and oracle/counts.py against what the paper and SPEC fix.

* SPEC worked examples (tests/golden/spec_mask_examples.json)
* section partition / triangle identity
* closed forms vs brute force, and vs the C oracle's own enumerator
* O(N) growth of the kept set
* the layer rule percentages of P:L409 (reading R2)
"""
import json
import os
import random

import numpy as np
import pytest

from oracle import counts, cref, masks

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _mask(kind, e):
    n = e["n"]
    if kind == "causal":
        return masks.causal_mask(n)
    if kind == "streaming":
        return masks.streaming_mask(n, e["si"], e["sl"])
    if kind == "last_qk":
        return masks.last_qk_mask(n, e["si"], e["sl"], e["last"])
    if kind == "middle_qk":
        return masks.middle_qk_mask(n, e["si"], e["sl"], e["last"])
    if kind == "triangle":
        return masks.triangle_mask(n, e["si"], e["sl"], e["last"])
    raise KeyError(kind)


def test_spec_worked_examples():
    ex = json.load(open(os.path.join(GOLD, "spec_mask_examples.json")))["examples"]
    assert len(ex) >= 10
    for e in ex:
        assert masks.popcount(_mask(e["kind"], e)) == e["popcount"], e


def test_empty_sequence_rejected():
    with pytest.raises(ValueError):
        masks.causal_mask(0)


def test_partition_and_triangle_identity_exhaustive():
    """Streaming, Middle and Last sections are disjoint and cover M."""
    rng = random.Random(1)
    for _ in range(60):
        n = rng.randint(1, 40)
        si, sl, last = rng.randint(0, 6), rng.randint(1, 12), rng.randint(1, 12)
        c = masks.causal_mask(n)
        s = masks.streaming_mask(n, si, sl)
        lq = masks.last_qk_mask(n, si, sl, last)
        mq = masks.middle_qk_mask(n, si, sl, last)
        t = masks.triangle_mask(n, si, sl, last)
        assert not (s & lq).any() and not (s & mq).any() and not (lq & mq).any()
        assert np.array_equal(s | lq | mq, c)
        assert np.array_equal(t, c & ~mq)
        assert np.array_equal(t, s | lq)
        assert np.array_equal(masks.mask_vectorised(n, si, sl, last, False), t)
        assert np.array_equal(masks.mask_vectorised(n, si, sl, last, True), c)


def test_degenerate_params_equal_causal():
    """si+sl >= n or last >= n: middle empty, triangle == causal."""
    for n in (1, 5, 17):
        c = masks.causal_mask(n)
        assert np.array_equal(masks.triangle_mask(n, 0, n, 1), c)       # window >= N
        assert np.array_equal(masks.triangle_mask(n, 3, 2, n), c)       # last >= N
        assert np.array_equal(masks.triangle_mask(n, n, 1, 1), c)       # sink >= N


def test_diagonal_always_admitted():
    for n, si, sl, last in [(9, 0, 1, 1), (20, 2, 1, 3), (33, 0, 1, 1)]:
        t = masks.triangle_mask(n, si, sl, last)
        assert t.diagonal().all()


def test_closed_forms_vs_bruteforce():
    rng = random.Random(7)
    for _ in range(400):
        n = rng.randint(1, 80)
        si, sl, last = rng.randint(0, 10), rng.randint(1, 40), rng.randint(1, 40)
        bt = masks.popcount_bruteforce(n, si, sl, last)
        assert counts.triangle_pairs(n, si, sl, last) == bt
        assert counts.streaming_pairs(n, si, sl) == masks.popcount(masks.streaming_mask(n, si, sl))
        assert counts.last_section_pairs(n, si, sl, last) == masks.popcount(
            masks.last_qk_mask(n, si, sl, last))
        assert counts.dense_pairs(n) == masks.popcount_bruteforce(n, si, sl, last, dense=True)


def test_closed_form_vs_c_enumerator():
    """The C oracle's literal predicate agrees with the closed form at larger n."""
    for n, si, sl, last in [(512, 4, 64, 64), (3000, 8, 512, 128), (4097, 8, 512, 128),
                            (700, 0, 1, 1), (1000, 16, 100, 900)]:
        assert cref.pair_count(n, si, sl, last, False) == counts.triangle_pairs(n, si, sl, last)
        assert cref.pair_count(n, si, sl, last, True) == counts.dense_pairs(n)


def test_linear_growth():
    """count(2n)/count(n) <= 2.25 for n >= 4(si+sl+last)."""
    for si, sl, last in [(8, 512, 128), (4, 64, 64), (64, 128, 128)]:
        n0 = 4 * (si + sl + last)
        for n in (n0, 2 * n0, 8192, 32768, 131072):
            if n < n0:
                continue
            r = counts.triangle_pairs(2 * n, si, sl, last) / counts.triangle_pairs(n, si, sl, last)
            assert r <= 2.25
            assert counts.dense_pairs(2 * n) / counts.dense_pairs(n) > 3.9


def test_streaming_monotone():
    for n in (10, 33):
        prev = -1
        for si in range(0, 8):
            c = counts.streaming_pairs(n, si, 3)
            assert c >= prev
            prev = c


def test_layer_rule_percentages():
    g = json.load(open(os.path.join(GOLD, "paper_layer_rule.json")))
    for c in g["cases"]:
        tri = sum(not masks.layer_is_dense(l, c["tri_start"]) for l in range(c["n_layers"]))
        assert round(100.0 * tri / c["n_layers"], 1) == c["triangle_fraction_pct"]
    # and the paper's own configuration: Llama 16 dense + 16 triangle
    h = json.load(open(os.path.join(GOLD, "paper_hparams.json")))
    assert sum(masks.layer_is_dense(l, h["tri_start"]["llama-3.1-8b"]) for l in range(32)) == 16
    assert sum(not masks.layer_is_dense(l, h["tri_start"]["qwen2.5-7b"]) for l in range(28)) == 8
