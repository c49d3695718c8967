"""TriangleMix oracle -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

A plain, slow, obviously correct CPU implementation of what the TriangleMix
prefill-attention hot path computes (arxiv 2507.21526).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import, call, link or execute anything under
``oracle/``.  The product path (``paper_2507_21526_b200``) never imports it
and shares no code, header, table or helper with it.

Modules
-------
masks      the mask predicates of PAPER.md section 2.1/2.2/2.4 written out
           literally (0-based reading, R1), brute-force popcounts,
           and the per-layer dense/triangle rule (R2).
counts     closed-form kept-pair counts (derived from the predicates; pinned
           against brute force in tests).
textbook   NumPy fp64: the full N x N score matrix with -inf fill, literally
           A' = Softmax(QK^T/sqrt(d) - c(1-M')), c -> +inf.
cref       ctypes loader for attn_oracle.c: plain C fp64 two-pass masked
           softmax, one (head,row) at a time, OpenMP over rows.
schedule_ref  independent enumerator of the static block schedule spec in
           DESIGN.md section 4 (the byte format the C-ABI exports).

Every function cites the PAPER.md line (P:Lnnn) or SPEC.md line (S:Lnnn) it
follows.  Parity pins live in tests/test_oracle_*.py.
"""
