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
NAMES = {7: "MM.waitP_B", 8: "MM.waitP_A", 9: "MM.waitV", 18: "MM.waitK", 19: "MM.gotK", 1: "PR.Q", 2: "PR.K", 3: "PR.V", 10: "MM.gotP_A", 11: "MM.PV_A", 12: "MM.QK_A", 13: "MM.gotP_B",
         14: "MM.PV_B", 15: "MM.QK_B", 16: "MM.gotQ", 17: "MM.gotV", 20: "SM.gotS", 21: "SM.Pdone",
         22: "SM.epi0", 23: "SM.epi1", 24: "SM.ldS", 25: "SM.max", 26: "SM.exp", 27: "SM.epiO", 30: "EP.waitA", 31: "EP.waitB", 32: "EP.gotA", 33: "EP.gotB", 34: "EP.doneA", 35: "EP.doneB"}
for cta in (0, 77):
    os.environ["TA_TRACE_CTA"] = str(cta)
    for _ in range(2):
        if dense:
            ta.dense_attn_prefill(q, k, v)
        else:
            ta.triangle_attn_prefill(q, k, v, sink=c.si, window=c.sl, last_q=c.last)
    torch.cuda.synchronize()
    buf = np.zeros(5 * 65536, dtype=np.uint64)
    lib.ta_debug_trace_read(buf.ctypes.data, buf.nbytes)
    ev = []
    for role in range(5):
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
    for role in (2, 3):
        seq = {cd: [t for t, r, c2, a in ev if r == role and c2 == cd] for cd in (20, 24, 25, 26, 21)}
        n = min(len(v) for v in seq.values())
        if n:
            st = [np.median(np.array(seq[b][:n]) - np.array(seq[a][:n])) for a, b in ((20, 24), (24, 25), (25, 26), (26, 21))]
            print(f"softmax {'AB'[role-2]} phases (median): ldS {st[0]:.0f}  max {st[1]:.0f}  exp {st[2]:.0f}  st/arrive {st[3]:.0f}")
    # MMA warp idle time by what it waits for (pairs of wait-start / wait-end events)
    mm = [(t, cd) for t, r, cd, a in ev if r == 1]
    waits = {"V": 0, "K": 0, "P_A": 0, "P_B": 0}
    pairs = {9: (17, "V"), 18: (19, "K"), 8: (10, "P_A"), 7: (13, "P_B")}
    for i in range(len(mm) - 1):
        t, cd = mm[i]
        if cd in pairs:
            end_cd, nm = pairs[cd]
            for t2, cd2 in mm[i + 1:i + 4]:
                if cd2 == end_cd:
                    waits[nm] += t2 - t
                    break
    span = mm[-1][0] - mm[0][0]
    print("MMA warp wait fractions:", {k: round(v / span, 3) for k, v in waits.items()}, "span", span)
    # per item: MM.gotQ to next MM.gotQ, blocks = number of MM.gotV in between
    gq = [i for i, e in enumerate(ev) if e[1] == 1 and e[2] == 16]
    per = {}
    for a, b in zip(gq, gq[1:]):
        nb = sum(1 for e in ev[a:b] if e[1] == 1 and e[2] == 17)
        per.setdefault(nb, []).append(ev[b][0] - ev[a][0])
    if len(gq) > 6:
        a, b = gq[4], gq[6]
        print("--- events of two consecutive items (from MM.gotQ #4):")
        for t_, r_, cd_, a_ in ev[a - 20:b + 5]:
            lab = NAMES.get(cd_, str(cd_)) + ("(B)" if r_ == 3 else "(A)" if r_ == 2 else "")
            print(f"{t_ - ev[a][0]:9d} {lab:14s} {a_}")
    for nb in sorted(per):
        v = np.array(per[nb])
        print(f"items with {nb:4d} blocks: n={len(v):4d} median {np.median(v):8.0f} cycles = {np.median(v)/max(nb,1):7.0f}/block")
    ga = [t for t, r, cd, a in ev if r == 4 and cd == 32]; da = [t for t, r, cd, a in ev if r == 4 and cd == 34]
    gb = [t for t, r, cd, a in ev if r == 4 and cd == 33]; db = [t for t, r, cd, a in ev if r == 4 and cd == 35]
    if ga and da:
        n = min(len(ga), len(da)); m = min(len(gb), len(db))
        print("epilogue tile work (median cycles): A", np.median(np.array(da[:n]) - np.array(ga[:n])),
              "B", np.median(np.array(db[:m]) - np.array(gb[:m])))
    pvA = [t for t, r, cd, a in ev if r == 1 and cd == 10]
    doneA = [t for t, r, cd, a in ev if r == 2 and cd == 21]
    n = min(len(pvA), len(doneA))
    print("P_A arrive -> MMA sees it: med", np.median(np.array(pvA[:n]) - np.array(doneA[:n])))
