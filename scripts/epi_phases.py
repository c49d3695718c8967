import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
os.environ.setdefault("TA_LIBRARY", os.path.join(os.getcwd(), "paper_2507_21526_b200", "libtriattn_trace.so"))
import torch
import paper_2507_21526_b200 as ta
import synth
c = synth.CONFIGS["C3"]
q, k, v = (t.cuda() for t in synth.config_qkv(c, 16))
lib = ta._load()
lib.ta_debug_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
for _ in range(2):
    ta.triangle_attn_prefill(q, k, v, sink=c.si, window=c.sl, last_q=c.last)
torch.cuda.synchronize()
buf = np.zeros(8 * 65536, dtype=np.uint64)
lib.ta_debug_trace_read(buf.ctypes.data, buf.nbytes)
seg = buf[4 * 65536:5 * 65536]
seg = seg[seg != 0]
ev = [(int(w) & 0xffffffffffff, int(w) >> 56) for w in seg]
# tiles: gotX (32/33) then 40,42,44,41,43,45, done (34/35)
out = {}
cur = None
for t, cd in ev:
    if cd in (32, 33):
        cur = {"got": t}
    elif cur is not None:
        cur[cd] = t
        if cd in (34, 35):
            if all(x in cur for x in (40, 42, 44, 41, 43, 45)):
                seq = [cur["got"], cur[40], cur[42], cur[44], cur[41], cur[43], cur[45], t]
                out.setdefault("d", []).append(np.diff(seq))
            cur = None
d = np.array(out["d"])
print("tiles", len(d))
print("median phases: ld+pack h0, waitread+bar h0, sts+store h0, ld+pack h1, waitread+bar h1, sts+store h1, tail")
print(np.median(d, axis=0))
print("mean", d.mean(axis=0).round(0))
