"""Per-item cost of STREAM items in SM cycles (TA_CTA_CLOCK build): C3 shape, StreamingMix
(last_q = 0, so every item is a STREAM item), window sl in {256, 512, 1024, 2048}; mean
CTA cycles / items per CTA against S columns per item gives the per-item intercept and
the per-128-column slope."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2507_21526_b200 as ta  # noqa: E402

lib = ta._load()
lib.ta_debug_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
n, hq, hkv = 131072, 32, 8
g = torch.Generator(device="cuda").manual_seed(1)
q = torch.randn(hq, n, 128, device="cuda", generator=g).to(torch.bfloat16)
k = torch.randn(hkv, n, 128, device="cuda", generator=g).to(torch.bfloat16)
v = torch.randn(hkv, n, 128, device="cuda", generator=g).to(torch.bfloat16)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
items = hkv * (n // 64) / 148
rows = []
for sl in (256, 512, 1024, 2048):
    cyc = []
    for r in range(5):
        flush.zero_()
        ta.triangle_attn_prefill(q, k, v, sink=8, window=sl, last_q=0)
        torch.cuda.synchronize()
        buf = np.zeros(148, dtype=np.uint64)
        lib.ta_debug_trace_read(buf.ctypes.data, buf.nbytes)
        if r >= 2:
            cyc.append(float(buf.mean()))
    cols = 16 + ((sl + 63 - 112 + 127) // 128) * 128 + 112  # rough S columns per item
    per_item = float(np.median(cyc)) / items
    rows.append((sl, per_item))
    print(f"sl={sl}: mean CTA cycles {np.median(cyc):.0f}, per item {per_item:.0f}", flush=True)
x = np.array([r[0] for r in rows], dtype=float)
y = np.array([r[1] for r in rows])
b, a = np.polyfit(x, y, 1)
print(f"fit: per item = {a:.0f} + {b * 128:.0f} per 128 window keys")
