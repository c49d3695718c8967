"""Per-CTA item timeline at a kv-head shard shape (TA_TRACE build, clock64 cycles): startup
(kernel entry -> first Q / first S), every item's span and block count, and the drain after
the last item -- where a small shard's per-CTA time goes.

    TA_LIBRARY=paper_2507_21526_b200/libtriattn_trace.so python scripts/trace_shard.py [HQ HKV N]"""
import ctypes
import os
import sys

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, root)
os.environ.setdefault("TA_LIBRARY", os.path.join(root, "paper_2507_21526_b200", "libtriattn_trace.so"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2507_21526_b200 as ta  # noqa: E402
import synth  # noqa: E402

hq, hkv, n = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (4, 1, 32768)
q, k, v = (t.cuda() for t in synth.make_qkv(hq, hkv, n, 128, seed=3))
lib = ta._load()
lib.ta_debug_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for cta in (0, 37, 74, 111, 147):
    os.environ["TA_TRACE_CTA"] = str(cta)
    for _ in range(2):
        flush.zero_()
        ta.triangle_attn_prefill(q, k, v, sink=8, window=512, last_q=128)
    torch.cuda.synchronize()
    buf = np.zeros(8 * 65536, dtype=np.uint64)
    lib.ta_debug_trace_read(buf.ctypes.data, buf.nbytes)
    ev = []
    for role in range(8):
        seg = buf[role * 65536:(role + 1) * 65536]
        for w in seg[seg != 0]:
            w = int(w)
            ev.append((w & 0xffffffffffff, role, w >> 56, (w >> 48) & 0xff))
    ev.sort()
    t0 = ev[0][0]
    gq = [t - t0 for t, r, c, a in ev if r == 1 and c == 16]          # MMA: item's Q tiles ready
    gs = [t - t0 for t, r, c, a in ev if r == 2 and c == 20]          # softmax A: S ready
    pv = [(t - t0, a) for t, r, c, a in ev if r == 1 and c == 10]     # MMA: P ready (block a)
    epa = [t - t0 for t, r, c, a in ev if r == 4 and c == 34]         # epilogue done A
    epb = [t - t0 for t, r, c, a in ev if r == 4 and c == 35]         # epilogue done B
    print(f"== CTA {cta}: span {ev[-1][0] - t0} cycles; first Q {gq[0] if gq else -1}, first S(A) "
          f"{gs[0] if gs else -1}, last epilogue {max(epb) if epb else -1}")
    # item boundaries from the MMA's per-item Q waits; block counts from P-ready events
    bounds = gq + [ev[-1][0] - t0]
    for i in range(len(gq)):
        nb = sum(1 for t, a in pv if bounds[i] <= t < bounds[i + 1])
        print(f"   item {i}: starts {bounds[i]:8d}  span {bounds[i + 1] - bounds[i]:7d}  blocks {nb}")
