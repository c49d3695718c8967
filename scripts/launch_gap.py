"""Where the per-launch time outside the CTAs goes at a small shard (8-way C2: Hq 4, Hkv 1,
N 32K): library-event attention time (a) after an L2 flush (a 512 MiB memset kernel, as in
bench.py), (b) right after another attention call, (c) after a large-smem cuBLAS GEMM (what
precedes attention in a real layer: the QKV projection)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_21526_b200 as ta  # noqa: E402
import synth  # noqa: E402

hq, hkv, n = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (4, 1, 32768)
q, k, v = (t.cuda() for t in synth.make_qkv(hq, hkv, n, 128, seed=3))
o = torch.empty_like(q)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
a = torch.randn(8192, 4096, device="cuda", dtype=torch.bfloat16)
b = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)


def attn():
    ta.triangle_attn_prefill(q, k, v, o, sink=8, window=512, last_q=128)


for _ in range(5):
    attn()
torch.cuda.synchronize()
for name, pre in (("after_flush", lambda: flush.zero_()), ("after_attention", attn),
                  ("after_gemm", lambda: torch.mm(a, b))):
    res = []
    for _ in range(20):
        pre()
        ta.profile_begin()
        attn()
        pr = ta.profile_end()
        res.append(pr["attn_ms"] * 1e3)
    print(name, "attention kernel (library events) us: median %.1f" % statistics.median(res), flush=True)
