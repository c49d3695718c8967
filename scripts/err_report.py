"""Max / mean abs error against the oracle for the parity distributions (one library build:
TA_LIBRARY selects it).  Used to compare numerics of kernel variants."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2507_21526_b200 as ta, synth
from oracle import cref
for dist in ("iid", "large", "sink"):
    q, k, v = synth.make_qkv(32, 8, 4097, 128, 7, dist, 8)
    dev = torch.device('cuda')
    o = ta.triangle_attn_prefill(q.to(dev), k.to(dev), v.to(dev), sink=8, window=512, last_q=128)
    torch.cuda.synchronize()
    ref, _, _ = cref.attention(q, k, v, 8, 512, 128, False)
    e = np.abs(o.float().cpu().double().numpy() - ref)
    print(f"{dist:6s} max {e.max():.3e} mean {e.mean():.3e}", flush=True)
