"""One C3 triangle call after two warm-ups (for ncu metric captures of a kernel variant;
TA_LIBRARY selects the build, CFG the synth config, MODE=dense for the dense layer)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2507_21526_b200 as ta  # noqa: E402
import synth  # noqa: E402
c = synth.CONFIGS[os.environ.get("CFG", "C3")]
g = torch.Generator(device="cuda").manual_seed(1)
q = torch.randn(c.hq, c.n, c.d, device="cuda", generator=g).to(torch.bfloat16)
k = torch.randn(c.hkv, c.n, c.d, device="cuda", generator=g).to(torch.bfloat16)
v = torch.randn(c.hkv, c.n, c.d, device="cuda", generator=g).to(torch.bfloat16)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    flush.zero_()
    if os.environ.get("MODE") == "dense":
        ta.dense_attn_prefill(q, k, v)
    else:
        ta.triangle_attn_prefill(q, k, v, sink=c.si, window=c.sl, last_q=c.last)
torch.cuda.synchronize()
