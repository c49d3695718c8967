"""Debug: per-event timeline of one CTA from the TA_TRACE build (clock64 cycles)."""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("TA_LIBRARY", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                 "paper_2507_21526_b200", "libtriattn_trace.so"))
import torch
import paper_2507_21526_b200 as ta
import synth

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
dense = len(sys.argv) > 2 and sys.argv[2] == "dense"
c = synth.CONFIGS[name]
q, k, v = (t.cuda() for t in synth.config_qkv(c, 16))
lib = ta._load()
lib.ta_debug_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
NAMES = {1: "PR.Q", 2: "PR.K", 3: "PR.V", 16: "MM.gotQ", 9: "MM.waitV", 17: "MM.gotV", 8: "MM.waitP",
         10: "MM.gotP", 11: "MM.PV", 18: "MM.waitK", 19: "MM.gotK", 12: "MM.QK", 20: "SM.gotS", 21: "SM.end",
         24: "SM.ldS", 25: "SM.max", 26: "SM.exp", 27: "SM.waitPf", 28: "SM.gotPf", 29: "SM.waitS",
         30: "EP.waitA", 31: "EP.waitB", 32: "EP.gotA", 33: "EP.gotB", 34: "EP.doneA", 35: "EP.doneB"}
for cta in (0,):
    os.environ["TA_TRACE_CTA"] = str(cta)
    for _ in range(2):
        if dense:
            ta.dense_attn_prefill(q, k, v)
        else:
            ta.triangle_attn_prefill(q, k, v, sink=c.si, window=c.sl, last_q=c.last)
    torch.cuda.synchronize()
    buf = np.zeros(8 * 65536, dtype=np.uint64)
    lib.ta_debug_trace_read(buf.ctypes.data, buf.nbytes)
    ev = []
    for role in range(8):
        seg = buf[role * 65536:(role + 1) * 65536]
        seg = seg[seg != 0]
        for w in seg:
            w = int(w)
            code, arg, t = w >> 56, (w >> 48) & 0xff, w & 0xffffffffffff
            ev.append((t, role, code, arg))
    ev.sort()
    t0 = ev[0][0]
    print(f"=== CTA {cta}: {len(ev)} events, span {ev[-1][0]-t0} cycles")
    for t, role, code, arg in ev[:160]:
        lab = NAMES.get(code, str(code)) + ("" if role != 3 else "(B)") + ("(A)" if role == 2 else "")
        print(f"{t - t0:9d} {lab:14s} {arg}")
    # per-block statistics for softmax A/B
    for role in (2, 3):
        got = [t for t, r, cd, a in ev if r == role and cd == 20]
        done = [t for t, r, cd, a in ev if r == role and cd == 21]
        n = min(len(got), len(done))
        d = np.array(done[:n]) - np.array(got[:n])
        gap = np.array(got[1:n]) - np.array(done[:n - 1])
        print(f"softmax {'AB'[role-2]}: blocks={n} compute med={np.median(d):.0f} mean={d.mean():.0f}; "
              f"wait-for-S med={np.median(gap):.0f} mean={gap.mean():.0f}")
        wp = [t for t, r, cd, a in ev if r == role and cd == 27]
        gp = [t for t, r, cd, a in ev if r == role and cd == 28]
        m = min(len(wp), len(gp))
        if m:
            w = np.array(gp[:m]) - np.array(wp[:m])
            print(f"   P-buffer wait: lo med {np.median(w[0::2]):.0f} mean {w[0::2].mean():.0f}; hi med {np.median(w[1::2]):.0f} mean {w[1::2].mean():.0f}")
        ws = [t for t, r, cd, a in ev if r == role and cd == 29]
        m = min(len(ws), len(got))
        if m:
            print(f"   s_full wait: med {np.median(np.array(got[:m]) - np.array(ws[:m])):.0f}; end->waitS med {np.median(np.array(ws[1:m]) - np.array(done[:m-1])):.0f}")
        seq = {cd: [t for t, r, c2, a in ev if r == role and c2 == cd] for cd in (20, 24, 25, 26, 21)}
        n = min(len(vv) for vv in seq.values())
        if n:
            st = [np.median(np.array(seq[b_][:n]) - np.array(seq[a_][:n])) for a_, b_ in ((20, 24), (24, 25), (25, 26), (26, 21))]
            print(f"softmax {'AB'[role-2]} phases (median): ldS {st[0]:.0f}  max {st[1]:.0f}  exp {st[2]:.0f}  tail {st[3]:.0f}")
    gq = [i for i, e in enumerate(ev) if e[1] == 1 and e[2] == 16]
    if len(gq) > 6:
        a, b = gq[4], gq[6]
        print("--- events of two consecutive items (from MM.gotQ #4):")
        for t_, r_, cd_, a_ in ev[a - 20:b + 5]:
            lab = NAMES.get(cd_, str(cd_)) + ("(B)" if r_ == 3 else "(A)" if r_ == 2 else "")
            print(f"{t_ - ev[a][0]:9d} {lab:14s} {a_}")
    per = {}
    for a, b in zip(gq, gq[1:]):
        nb = sum(1 for e in ev[a:b] if e[1] == 1 and e[2] == 10)
        per.setdefault(nb, []).append(ev[b][0] - ev[a][0])
    for nb in sorted(per):
        vv = np.array(per[nb])
        print(f"items with {nb:4d} blocks: n={len(vv):4d} median {np.median(vv):8.0f} cycles = {np.median(vv)/max(nb,1):7.0f}/block")
    ga = [t for t, r, cd, a in ev if r == 4 and cd == 32]; da = [t for t, r, cd, a in ev if r == 4 and cd == 34]
    gb = [t for t, r, cd, a in ev if r == 4 and cd == 33]; db = [t for t, r, cd, a in ev if r == 4 and cd == 35]
    if ga and da:
        n = min(len(ga), len(da)); m = min(len(gb), len(db))
        print("epilogue tile work (median cycles): A", np.median(np.array(da[:n]) - np.array(ga[:n])),
              "B", np.median(np.array(db[:m]) - np.array(gb[:m])))

# drift across the four warps of tile A: per block, spread of "end" (and gotS) times
for code, nm in ((20, "gotS"), (21, "end")):
    per = [[t for t, r, cd, a in ev if r == rr and cd == code] for rr in (2, 5, 6, 7)]
    m = min(len(x) for x in per)
    if m:
        arr = np.array([x[:m] for x in per], dtype=np.float64)
        spread = arr.max(0) - arr.min(0)
        slow = np.bincount(arr.argmax(0), minlength=4)
        print(f"tile A warps {nm}: spread med {np.median(spread):.0f} mean {spread.mean():.0f}; slowest warp counts {slow.tolist()}")
