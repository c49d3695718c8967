"""One tiny triangle call (1 head, N = 64) repeated: for ncu's per-launch durations."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2507_21526_b200 as ta  # noqa: E402
import synth  # noqa: E402
q, k, v = (t.cuda() for t in synth.make_qkv(1, 1, 64, 128, seed=1))
for _ in range(8):
    ta.dense_attn_prefill(q, k, v)
    ta.triangle_attn_prefill(q, k, v)
torch.cuda.synchronize()
