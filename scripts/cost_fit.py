"""Calibrate the schedule's cost model from measured per-CTA SM cycles (TA_CTA_CLOCK build):
least-squares fit of  cycles_c = a * STREAM items_c + b * LASTQ 128-key blocks_c
+ c * LASTQ pieces_c + d  over the 148 CTAs of a triangle layer, and of the cost model's own
prediction (sum of item costs in columns) against the same cycles.

    TA_LIBRARY=variants/clk_base.so python scripts/cost_fit.py C3 C2 C4b"""
import ctypes
import os
import sys

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, root)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2507_21526_b200 as ta  # noqa: E402
import synth  # noqa: E402
from oracle import schedule_ref  # noqa: E402

lib = ta._load()
lib.ta_debug_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
sms = torch.cuda.get_device_properties(0).multi_processor_count
rows = []
for name in sys.argv[1:] or ["C3"]:
    c = synth.CONFIGS[name]
    for P in (1, 8):
        hq, hkv = c.hq // P if c.hkv >= P else c.hq, max(1, c.hkv // P)
        q, k, v = (t.cuda() for t in synth.make_qkv(hq, hkv, c.n, c.d, seed=7))
        cyc = []
        for r in range(4):
            flush.zero_()
            ta.triangle_attn_prefill(q, k, v, sink=c.si, window=c.sl, last_q=c.last)
            torch.cuda.synchronize()
            buf = np.zeros(sms, dtype=np.uint64)
            lib.ta_debug_trace_read(buf.ctypes.data, buf.nbytes)
            if r:
                cyc.append(buf.astype(np.float64))
        cyc = np.median(np.array(cyc), axis=0)
        hdr, items = schedule_ref.parse(ta.schedule_export(c.n, hq, hkv, c.d, sms, c.si, c.sl, c.last))
        geo = schedule_ref.geometry(c.n, hq, hkv, c.d, c.si, c.sl, c.last, False)
        X, model = [], []
        for cta in range(sms):
            its = items[off[cta]:off[cta + 1]]
            ns = sum(1 for it in its if it[0] == schedule_ref.STREAM)
            lq = [it for it in its if it[0] == schedule_ref.LASTQ]
            nb = sum(-(-(it[4] - it[3]) // 128) for it in lq)
            X.append([ns, nb, len(lq), 1.0])
            model.append(sum(schedule_ref.cost(geo, it) for it in its))
        X, model = np.array(X, dtype=np.float64), np.array(model, dtype=np.float64)
        coef, *_ = np.linalg.lstsq(X, cyc, rcond=None)
        pred = X @ coef
        r_model = np.corrcoef(model, cyc)[0, 1]
        print(f"{name} x{P}: cycles max {cyc.max():.0f} mean {cyc.mean():.0f} (max/mean {cyc.max() / cyc.mean():.4f}); "
              f"fit: STREAM item {coef[0]:.0f}, LASTQ block {coef[1]:.0f}, LASTQ piece {coef[2]:.0f}, "
              f"fixed {coef[3]:.0f} cycles (rms resid {np.sqrt(np.mean((pred - cyc) ** 2)):.0f}); "
              f"cost model vs cycles corr {r_model:.3f}; slowest CTA: {X[cyc.argmax()][:3].tolist()}",
              flush=True)
        if os.environ.get("DUMP"):
            order = np.argsort(cyc)
            for cta in list(order[:4]) + list(order[-6:]):
                its = items[off[cta]:off[cta + 1]]
                ps = sorted(it[2] for it in its if it[0] == schedule_ref.STREAM)
                short = sum(1 for it in its if it[0] == schedule_ref.STREAM
                            and schedule_ref.item_blocks(geo, it)[-1][2] <= 80)
                print(f"   cta {cta:3d} cycles {cyc[cta]:9.0f} model {model[cta]:7.0f} stream {X[cta][0]:.0f} "
                      f"(short-last {short}) lastq blocks {X[cta][1]:.0f} pieces {X[cta][2]:.0f} "
                      f"pairs {ps[:3]}..{ps[-2:]}")
        del q, k, v
