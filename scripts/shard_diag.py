"""Strong-scaling diagnosis on one GPU: for the per-rank shard shapes of C3 / C2 (P = 1, 2,
4, 8 kv-head shards) report the step time (outer CUDA events, PDL active), the attention
and merge kernel times (library events), and -- with TA_LIBRARY pointing at a TA_CTA_CLOCK
build -- the max and mean per-CTA SM cycles of the attention kernel."""
import ctypes
import json
import os
import sys

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, root)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2507_21526_b200 as ta  # noqa: E402
import synth  # noqa: E402

clock = "clk_" in os.environ.get("TA_LIBRARY", "")
lib = ta._load()
if clock:
    lib.ta_debug_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
names = sys.argv[1:] or ["C3", "C2"]
for name in names:
    c = synth.CONFIGS[name]
    for P in (1, 2, 4, 8):
        hq, hkv = c.hq // P, c.hkv // P
        q, k, v = (t.cuda() for t in synth.make_qkv(hq, hkv, c.n, c.d, seed=100 + P))
        o = torch.empty_like(q)

        def fn():
            ta.triangle_attn_prefill(q, k, v, o, sink=c.si, window=c.sl, last_q=c.last)
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        evs = []
        for _ in range(10):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            evs.append((a, b))
        torch.cuda.synchronize()
        step = float(np.median([a.elapsed_time(b) for a, b in evs]))
        ta.profile_begin()
        for _ in range(10):
            flush.zero_()
            fn()
        torch.cuda.synchronize()
        pr = ta.profile_end()
        row = {"cfg": name, "P": P, "step_ms": step, "attn_ms": pr["attn_ms"] / 10,
               "merge_ms": pr["merge_ms"] / 10}
        if clock:
            flush.zero_()
            fn()
            torch.cuda.synchronize()
            full = np.zeros(256 + 2 * 148, dtype=np.uint64)
            lib.ta_debug_trace_read(full.ctypes.data, full.nbytes)
            buf = full[:148]
            g = full[256:].reshape(148, 2).astype(np.int64)  # zeros unless a TA_GT build
            t0 = g[:, 0].min()
            # CTA start skew and end spread (globaltimer, us): launch ramp and tail
            row["cta_start_us_max"] = float((g[:, 0].max() - t0) / 1e3)
            row["cta_end_us_min"] = float((g[:, 1].min() - t0) / 1e3)
            row["cta_end_us_max"] = float((g[:, 1].max() - t0) / 1e3)
            span = (g[:, 1] - g[:, 0])[int(buf.argmax())]
            row["sm_mhz_est"] = float(buf.max() / (span / 1e3)) if span > 0 else None
            row["cta_cycles_max"] = int(buf.max())
            row["cta_cycles_mean"] = float(buf.mean())
            row["cta_cycles_min"] = int(buf.min())
        print(json.dumps(row), flush=True)
        del q, k, v, o
