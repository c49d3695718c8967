"""Wait accounting of a TA_WAITSTAT (+TA_CTA_CLOCK) build: mean over CTAs of the cycles each
role spends in each barrier wait, as a fraction of the CTA's elapsed cycles.
    TA_LIBRARY=variants/clk_ws.so python scripts/waitstat.py [C3|C2|...] [dense]"""
import ctypes
import os
import sys

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, root)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2507_21526_b200 as ta  # noqa: E402
import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
dense = len(sys.argv) > 2 and sys.argv[2] == "dense"
c = synth.CONFIGS[cfg]
q, k, v = (t.cuda() for t in synth.config_qkv(c, 16))
lib = ta._load()
lib.ta_debug_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    flush.zero_()
    if dense:
        ta.dense_attn_prefill(q, k, v)
    else:
        ta.triangle_attn_prefill(q, k, v, sink=c.si, window=c.sl, last_q=c.last)
torch.cuda.synchronize()
buf = np.zeros(4096 + 128 * 148, dtype=np.uint64)
lib.ta_debug_trace_read(buf.ctypes.data, buf.nbytes)
tot = buf[:148].astype(np.float64)
ws = buf[4096:].reshape(148, 8, 16)[:, :5, :].astype(np.float64)
names = {0: ("TMA", ["q_empty", "kv_empty"]),
         1: ("MMA", ["q_full", "kv_full V", "kv_full K(next)", "p_ready A", "p_hi A", "o_free", "p_ready B",
                     "p_hi B", "issue QK", "issue PV", "commits", "next item_info"]),
         2: ("softmax A", ["s_full", "o_free (publish)"]),
         3: ("softmax B", ["s_full", "o_free (publish)"]),
         4: ("epilogue", ["l_ready", "o_full", "staging TMA read", "staging bar.sync"])}
print(f"{cfg} {'dense' if dense else 'triangle'}: CTA cycles mean {tot.mean():.0f} max {tot.max():.0f}")
for role, (nm, ks) in names.items():
    parts = [f"{k_}: {100 * (ws[:, role, i] / tot).mean():.1f}%" for i, k_ in enumerate(ks)]
    print(f"  {nm:10s} " + "  ".join(parts))
bp, it = ws[:, 1, 14].mean(), ws[:, 1, 15].mean()
print(f"  MMA: {bp:.0f} block pairs and {it:.0f} items per CTA; {tot.mean() / max(bp, 1):.0f} cycles per block pair; "
      f"issue per block pair: QK {ws[:, 1, 8].mean() / max(bp, 1):.0f}, PV {ws[:, 1, 9].mean() / max(bp, 1):.0f}, "
      f"commits {ws[:, 1, 10].mean() / max(bp, 1):.0f} cycles")
