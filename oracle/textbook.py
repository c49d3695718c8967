"""Textbook masked softmax attention in NumPy fp64.  TEST INFRASTRUCTURE.

Literally P:L104-118 (section 2.1):

    A' = Softmax( QK^T / sqrt(d) - c (1 - M') ),   O = A' V

with c -> +inf (reading R3: masked scores are excluded, set to -inf before the
row softmax), the full N x N score matrix materialised, and GQA head mapping
h -> floor(h / (Hq/Hkv)) (reading R13).  Intended for N <= ~4096.
"""
from __future__ import annotations

import numpy as np

from . import masks


def softmax_rows(s: np.ndarray) -> np.ndarray:
    """Row softmax with max subtraction; -inf entries get weight exactly 0."""
    m = np.max(s, axis=-1, keepdims=True)
    e = np.exp(s - m)
    return e / np.sum(e, axis=-1, keepdims=True)


def attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, mask: np.ndarray,
              scale: float | None = None):
    """Single head.  q,k,v: (N, d) float64; mask: (N, N) bool.  Returns (O, A, lse)."""
    n, d = q.shape
    if scale is None:
        scale = 1.0 / np.sqrt(d)
    s = (q @ k.T) * scale
    s = np.where(mask, s, -np.inf)
    a = softmax_rows(s)
    m = np.max(s, axis=-1)
    lse = m + np.log(np.sum(np.exp(s - m[:, None]), axis=-1))
    return a @ v, a, lse


def mha(q: np.ndarray, k: np.ndarray, v: np.ndarray, si: int, sl: int, last: int,
        dense: bool, scale: float | None = None):
    """GQA multi-head: q (Hq,N,d), k/v (Hkv,N,d) float64 -> O (Hq,N,d), lse (Hq,N)."""
    hq, n, d = q.shape
    hkv = k.shape[0]
    g = hq // hkv
    m = masks.mask_vectorised(n, si, sl, last, dense)
    o = np.empty((hq, n, d))
    lse = np.empty((hq, n))
    for h in range(hq):
        o[h], _, lse[h] = attention(q[h], k[h // g], v[h // g], m, scale)
    return o, lse
