"""Mask predicates of TriangleMix, written out from the paper.  TEST INFRASTRUCTURE.

Index convention (reading R1, adopted from SPEC S:L118-121): 0-based
query row i and key column j.  The paper's 1-based inequalities become

  sink      "j <= si"        ->  j <  si          (si sink keys)
  window    "i - j <= sl"    ->  i - j <  sl      (sl keys including the diagonal)
  last rows "N - i < last"   ->  i >= N - last    (last query rows)
  "j > si", "i - j > sl"     ->  j >= si, i - j >= sl   (their complements)

Everything here is deliberately literal and slow.
"""
from __future__ import annotations

import numpy as np


def causal(i: int, j: int, n: int) -> bool:
    """M_{i,j} of P:L104-110 (section 2.1): the standard causal mask, j <= i."""
    return 0 <= j <= i < n


def streaming(i: int, j: int, n: int, si: int, sl: int) -> bool:
    """M^streaming of P:L120-131 (section 2.1 eq.): i>=j and (j<=si or i-j<=sl), 0-based (R1)."""
    return causal(i, j, n) and (j < si or i - j < sl)


def last_qk(i: int, j: int, n: int, si: int, sl: int, last: int) -> bool:
    """M^last of P:L150-161 (section 2.2 eq.): i>=j, N-i<last, j>si, i-j>sl, 0-based (R1)."""
    return causal(i, j, n) and i >= n - last and j >= si and i - j >= sl


def middle_qk(i: int, j: int, n: int, si: int, sl: int, last: int) -> bool:
    """M^middle of P:L163-172 (section 2.2 eq.): i>=j, N-i>=last, j>si, i-j>sl, 0-based (R1)."""
    return causal(i, j, n) and i < n - last and j >= si and i - j >= sl


def triangle(i: int, j: int, n: int, si: int, sl: int, last: int) -> bool:
    """Deep-layer mask  M - M^middle  of P:L263-269 (section 2.4 eq.)."""
    return causal(i, j, n) and not middle_qk(i, j, n, si, sl, last)


def layer_is_dense(layer: int, tri_start: int) -> bool:
    """Per-layer pattern choice, P:L255-269 / P:L295, reading R2.

    Layers [0, tri_start) are dense, [tri_start, L) triangle.  Pinned by P:L409:
    tri_start=12 on 32 layers is "62.5% of the layers" triangle, tri_start=20 on
    Qwen's 28 layers is "28.6%".
    """
    return layer < tri_start


# ---------------------------------------------------------------- matrices
def _matrix(pred, n: int, *args) -> np.ndarray:
    m = np.zeros((n, n), dtype=bool)
    for i in range(n):
        for j in range(n):
            m[i, j] = pred(i, j, n, *args)
    return m


def causal_mask(n: int) -> np.ndarray:
    """N x N boolean causal mask.  Brute force; n <= a few thousand."""
    if n < 1:
        raise ValueError("EmptySequence (S:L56)")
    return _matrix(causal, n)


def streaming_mask(n: int, si: int, sl: int) -> np.ndarray:
    return _matrix(streaming, n, si, sl)


def last_qk_mask(n: int, si: int, sl: int, last: int) -> np.ndarray:
    return _matrix(last_qk, n, si, sl, last)


def middle_qk_mask(n: int, si: int, sl: int, last: int) -> np.ndarray:
    return _matrix(middle_qk, n, si, sl, last)


def triangle_mask(n: int, si: int, sl: int, last: int) -> np.ndarray:
    return _matrix(triangle, n, si, sl, last)


def mask_vectorised(n: int, si: int, sl: int, last: int, dense: bool) -> np.ndarray:
    """Same predicate as `triangle`/`causal`, evaluated with numpy broadcasting.

    Used by the textbook oracle for n up to ~4096 where the double Python loop
    is too slow; pinned element-for-element against the loop version in tests.
    """
    i = np.arange(n)[:, None]
    j = np.arange(n)[None, :]
    c = j <= i
    if dense:
        return c
    middle = c & (i < n - last) & (j >= si) & (i - j >= sl)
    return c & ~middle


def popcount(m: np.ndarray) -> int:
    """Exact number of admitted pairs."""
    return int(np.count_nonzero(m))


def popcount_bruteforce(n: int, si: int, sl: int, last: int, dense: bool = False) -> int:
    """Kept pairs per head by enumerating the literal predicate (no matrix)."""
    tot = 0
    for i in range(n):
        for j in range(i + 1):
            if dense or triangle(i, j, n, si, sl, last):
                tot += 1
    return tot


def row_keys(i: int, n: int, si: int, sl: int, last: int, dense: bool) -> list[int]:
    """J_i, the admitted key set of row i (SURVEY section 8(c) / P:L263-269)."""
    return [j for j in range(i + 1) if dense or triangle(i, j, n, si, sl, last)]
