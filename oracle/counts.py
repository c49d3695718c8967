"""Closed-form kept-pair counts.  TEST INFRASTRUCTURE.

Derived from the predicates in masks.py (reading R1),
with w = si + sl and R = max(0, N - last):

  streaming row i keeps  min(si, i+1) + |[max(si, i-sl+1), i]|  = min(i+1, w)
  last-section row i (i >= N-last) keeps  |[si, i-sl]| = max(0, i - sl - si + 1)
  triangle rows i >= N-last are full causal rows (M - M^middle, middle empty there)

so per head

  streaming(N)  = sum_{i<N} min(i+1, w)
                = N(N+1)/2                      if N <= w
                = w(w+1)/2 + (N-w) w             otherwise
  triangle(N)   = streaming(R) + N(N+1)/2 - R(R+1)/2
  dense(N)      = N(N+1)/2

These back the O(N) claim of P:L253 / P:L271 ("the elements in the Streaming and
Last Q-K sections grow only linearly with N").  Pinned against brute force in
tests/test_oracle_masks.py.
"""
from __future__ import annotations


def streaming_pairs(n: int, si: int, sl: int) -> int:
    w = si + sl
    if n <= w:
        return n * (n + 1) // 2
    return w * (w + 1) // 2 + (n - w) * w


def last_section_pairs(n: int, si: int, sl: int, last: int) -> int:
    """|M^last| = sum over the last rows of max(0, i - sl - si + 1)."""
    tot = 0
    for i in range(max(0, n - last), n):
        tot += max(0, i - sl - si + 1)
    return tot


def triangle_pairs(n: int, si: int, sl: int, last: int) -> int:
    r = max(0, n - last)
    return streaming_pairs(r, si, sl) + n * (n + 1) // 2 - r * (r + 1) // 2


def dense_pairs(n: int) -> int:
    return n * (n + 1) // 2


def kept_flops(n: int, hq: int, d: int, si: int, sl: int, last: int, dense: bool) -> int:
    """Algorithmic FLOPs: 2d (QK^T) + 2d (PV) per kept pair per q-head."""
    p = dense_pairs(n) if dense else triangle_pairs(n, si, sl, last)
    return 4 * d * hq * p
