"""Parity of each kernel variant (variants/clk_*.so) against the fp64 oracle on the stress
distributions at the Llama shape (Hq=32, Hkv=8, N=4097): max-abs / mean-abs per variant."""
import glob
import os
import subprocess
import sys

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, root)
    import numpy as np
    import torch
    import paper_2507_21526_b200 as ta
    import synth
    from oracle import cref
    out = []
    for dist in os.environ.get("DISTS", "iid,large,sink,ones_v,ramp").split(","):
        q, k, v = synth.make_qkv(32, 8, 4097, 128, 77, dist, 8)
        o = ta.triangle_attn_prefill(q.cuda(), k.cuda(), v.cuda(), sink=8, window=512, last_q=128)
        od = ta.dense_attn_prefill(q.cuda(), k.cuda(), v.cuda())
        torch.cuda.synchronize()
        ref, _, _ = cref.attention(q, k, v, 8, 512, 128, False)
        refd, _, _ = cref.attention(q, k, v, 0, 1, 1, True)
        e = np.abs(o.float().cpu().double().numpy() - ref)
        ed = np.abs(od.float().cpu().double().numpy() - refd)
        out.append(f"{dist}: tri {e.max():.2e}/{e.mean():.1e} dense {ed.max():.2e}/{ed.mean():.1e}")
    print(" | ".join(out))
    sys.exit(0)
sos = sys.argv[1:] or sorted(glob.glob(os.path.join(root, "variants", "clk_*.so")))
for so in sos:
    r = subprocess.run([sys.executable, __file__, "--child"], env=dict(os.environ, TA_LIBRARY=so),
                       capture_output=True, text=True)
    print(os.path.basename(so), r.stdout.strip() or r.stderr[-300:], flush=True)
