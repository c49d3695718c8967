"""Clock-independent, whole-kernel comparison of kernel variants: every variants/clk_*.so is a
TA_CTA_CLOCK build that records each CTA's elapsed SM cycles; the kernel's critical time is
the max over CTAs.  Runs C3 triangle (and dense with --dense) a few times per build,
interleaved, and reports the median of max-over-CTA cycles and the mean over CTAs."""
import ctypes, glob, os, subprocess, sys
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, root)
    import numpy as np, torch
    import paper_2507_21526_b200 as ta
    import synth
    cfg, dense, reps = sys.argv[2], sys.argv[3] == "1", int(sys.argv[4])
    c = synth.CONFIGS[cfg]
    q, k, v = (t.cuda() for t in synth.config_qkv(c, 16))
    lib = ta._load()
    lib.ta_debug_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    mx, mean = [], []
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda") if os.environ.get("FLUSH", "1") == "1" else None
    for r in range(reps + 2):
        if flush is not None:
            flush.zero_()  # same L2 state as bench.py's timed steps
        mode = os.environ.get("MODE", "")
        if dense:
            ta.dense_attn_prefill(q, k, v)
        elif mode == "last":    # f1: final-layer last rows only
            ta.last_rows_attn_prefill(q, k, v, last_q=c.last)
        elif mode == "smix":    # f3: StreamingMix layer (last_q = 0)
            ta.triangle_attn_prefill(q, k, v, sink=c.si, window=c.sl, last_q=0)
        else:
            ta.triangle_attn_prefill(q, k, v, sink=c.si, window=c.sl, last_q=c.last)
        torch.cuda.synchronize()
        buf = np.zeros(148, dtype=np.uint64)
        lib.ta_debug_trace_read(buf.ctypes.data, buf.nbytes)
        if r >= 2:
            mx.append(int(buf.max())); mean.append(float(buf.mean()))
    print(int(np.median(mx)), int(np.median(mean)))
    sys.exit(0)
cfg = os.environ.get("CFG", "C3")
dense = "--dense" in sys.argv
sos = sorted(glob.glob(os.path.join(root, "variants", "clk_*.so")))
res = {os.path.basename(s): [] for s in sos}
for rnd in range(3):
    for so in (sos if rnd % 2 == 0 else sos[::-1]):
        out = subprocess.run([sys.executable, __file__, "--child", cfg, "1" if dense else "0", "5"],
                             env=dict(os.environ, TA_LIBRARY=so), capture_output=True, text=True)
        try:
            a, b = out.stdout.split()
            res[os.path.basename(so)].append((int(a), int(b)))
        except Exception:
            res[os.path.basename(so)].append(out.stderr[-200:])
for k, v in res.items():
    ok = sorted(x for x in v if isinstance(x, tuple))
    print(k, "max-CTA cycles", [x[0] for x in ok], "mean-CTA", [x[1] for x in ok], flush=True)
