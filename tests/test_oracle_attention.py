"""Pins for the attention oracles (oracle/textbook.py, oracle/attn_oracle.c).

Each pin is something other than the oracle itself:
* brute force with Python math.exp on tiny inputs, iterating the admitted key
  set of the literal predicate (no numpy vectorisation, no matrix);
* a library routine: torch scaled_dot_product_attention(is_causal=True) in fp64
  on CPU for dense causal, and with enable_gqa for the GQA head mapping;
* special cases the paper/SPEC fix: N=1 -> O=V_0, V=1 -> O=1
  (S:L171), Q=0 -> uniform weights over J_i, window >= N -> dense
  causal, softmax rows sum to 1;
* the C oracle agrees with the textbook within 1e-12.
"""
import math
import random

import numpy as np
import pytest
import torch

import synth
from oracle import cref, masks, textbook


def _f64(t):
    return t.to(torch.float64).numpy()


def _bruteforce_row(q, k, v, i, n, si, sl, last, dense, scale):
    keys = masks.row_keys(i, n, si, sl, last, dense)
    s = [scale * sum(q[i, c] * k[j, c] for c in range(q.shape[1])) for j in keys]
    m = max(s)
    w = [math.exp(x - m) for x in s]
    tot = sum(w)
    return [sum(w[t] * v[keys[t], c] for t in range(len(keys))) / tot for c in range(v.shape[1])]


@pytest.mark.parametrize("dense", [False, True])
def test_textbook_and_c_vs_bruteforce_tiny(dense):
    rng = random.Random(3)
    for trial in range(6):
        n = rng.randint(1, 12)
        d = rng.choice([2, 4, 8])
        si, sl, last = rng.randint(0, 3), rng.randint(1, 4), rng.randint(1, 4)
        q, k, v = synth.make_qkv(2, 1, n, d, seed=100 + trial)
        qf, kf, vf = _f64(q), _f64(k), _f64(v)
        scale = 1.0 / math.sqrt(d)
        o_t, _ = textbook.mha(qf, kf, vf, si, sl, last, dense)
        o_c, _, _ = cref.attention(q, k, v, si, sl, last, dense)
        for h in range(2):
            for i in range(n):
                ref = _bruteforce_row(qf[h], kf[0], vf[0], i, n, si, sl, last, dense, scale)
                assert np.allclose(o_t[h, i], ref, atol=1e-13, rtol=0)
                assert np.allclose(o_c[h, i], ref, atol=1e-13, rtol=0)


def test_dense_equals_torch_sdpa_fp64():
    q, k, v = synth.make_qkv(4, 4, 200, 16, seed=5)
    ref = torch.nn.functional.scaled_dot_product_attention(
        q.double()[None], k.double()[None], v.double()[None], is_causal=True)[0].numpy()
    o_t, _ = textbook.mha(_f64(q), _f64(k), _f64(v), 0, 1, 1, dense=True)
    o_c, _, _ = cref.attention(q, k, v, 0, 1, 1, True)
    assert np.abs(o_t - ref).max() < 1e-12
    assert np.abs(o_c - ref).max() < 1e-12


def test_gqa_mapping_matches_sdpa_enable_gqa():
    """h -> h // (Hq/Hkv) (reading R13) is torch/Llama repeat_kv semantics."""
    q, k, v = synth.make_qkv(8, 2, 96, 16, seed=6)
    ref = torch.nn.functional.scaled_dot_product_attention(
        q.double()[None], k.double()[None], v.double()[None], is_causal=True,
        enable_gqa=True)[0].numpy()
    o_c, _, _ = cref.attention(q, k, v, 0, 1, 1, True)
    assert np.abs(o_c - ref).max() < 1e-12


def test_triangle_equals_sdpa_with_explicit_mask():
    """Triangle = SDPA with the boolean mask M - M^middle built from the section masks."""
    n, si, sl, last = 150, 3, 20, 17
    q, k, v = synth.make_qkv(2, 1, n, 32, seed=8)
    m = masks.causal_mask(n) & ~masks.middle_qk_mask(n, si, sl, last)
    ref = torch.nn.functional.scaled_dot_product_attention(
        q.double()[None], k.double()[None].expand(1, 2, n, 32),
        v.double()[None].expand(1, 2, n, 32), attn_mask=torch.from_numpy(m))[0].numpy()
    o_c, _, _ = cref.attention(q, k, v, si, sl, last, False)
    assert np.abs(o_c - ref).max() < 1e-12


def test_c_oracle_vs_textbook_random():
    rng = random.Random(11)
    for trial in range(8):
        hkv = rng.choice([1, 2])
        hq = hkv * rng.choice([1, 3, 4])
        n = rng.randint(1, 600)
        d = rng.choice([16, 64, 128])
        si, sl, last = rng.randint(0, 16), rng.randint(1, 200), rng.randint(1, 100)
        dense = rng.random() < 0.3
        q, k, v = synth.make_qkv(hq, hkv, n, d, seed=200 + trial, dist=rng.choice(
            ["iid", "large", "sink"]), si=si)
        o_t, lse_t = textbook.mha(_f64(q), _f64(k), _f64(v), si, sl, last, dense)
        o_c, lse_c, _ = cref.attention(q, k, v, si, sl, last, dense)
        assert np.abs(o_t - o_c).max() < 1e-12
        assert np.abs(lse_t - lse_c).max() < 1e-10


def test_row_subset_matches_full():
    q, k, v = synth.make_qkv(4, 2, 300, 64, seed=12)
    o, lse, _ = cref.attention(q, k, v, 8, 64, 32, False)
    rows = [0, 7, 150, 268, 299]
    o_s, lse_s, _ = cref.attention(q, k, v, 8, 64, 32, False, rows=rows)
    assert np.array_equal(o_s, o[:, rows])
    assert np.array_equal(lse_s, lse[:, rows])


def test_special_cases():
    # N = 1 -> O = V_0
    q, k, v = synth.make_qkv(3, 1, 1, 8, seed=1)
    o, _, _ = cref.attention(q, k, v, 8, 512, 128, False)
    assert np.array_equal(o[:, 0], np.repeat(_f64(v)[0, :1], 3, axis=0))
    # V = 1 -> O = 1 exactly up to rounding of the normalisation
    q, k, v = synth.make_qkv(2, 2, 257, 16, seed=2, dist="ones_v")
    o, _, _ = cref.attention(q, k, v, 4, 30, 20, False)
    assert np.abs(o - 1.0).max() < 1e-14
    # window >= N -> triangle == dense causal
    q, k, v = synth.make_qkv(2, 1, 100, 16, seed=3)
    a, _, _ = cref.attention(q, k, v, 2, 100, 1, False)
    b, _, _ = cref.attention(q, k, v, 0, 1, 1, True)
    assert np.array_equal(a, b)


def test_zero_q_onehot_v_is_exact_count_ratio():
    """Q = 0 -> uniform weights; with V[j, j mod d] = 1 the output is #{j in J_i: j = c mod d}/|J_i|."""
    n, d, si, sl, last = 300, 16, 5, 40, 30
    q, k, v = synth.make_qkv(1, 1, n, d, seed=4, dist="zeroq_onehot")
    o, _, _ = cref.attention(q, k, v, si, sl, last, False)
    for i in range(n):
        keys = masks.row_keys(i, n, si, sl, last, False)
        expect = np.zeros(d)
        for j in keys:
            expect[j % d] += 1
        expect /= len(keys)
        assert np.abs(o[0, i] - expect).max() < 1e-15


def test_softmax_rows_sum_to_one():
    n, si, sl, last = 64, 2, 8, 8
    q, k, v = synth.make_qkv(1, 1, n, 8, seed=9, dist="large")
    m = masks.triangle_mask(n, si, sl, last)
    _, a, _ = textbook.attention(_f64(q)[0], _f64(k)[0], _f64(v)[0], m)
    assert np.abs(a.sum(axis=1) - 1).max() < 1e-14
    assert (a[~m] == 0).all()
