"""Merge kernel time at C3 for each warps-per-row setting (TA_MERGE_W), library events."""
import os
import subprocess
import sys

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, root)
    import torch
    import paper_2507_21526_b200 as ta
    import synth
    c = synth.CONFIGS[sys.argv[2]]
    P = int(sys.argv[3])
    q, k, v = (t.cuda() for t in synth.make_qkv(c.hq // P, c.hkv // P, c.n, c.d, seed=3))
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        ta.triangle_attn_prefill(q, k, v)
    torch.cuda.synchronize()
    ta.profile_begin()
    for _ in range(20):
        flush.zero_()
        ta.triangle_attn_prefill(q, k, v)
    torch.cuda.synchronize()
    pr = ta.profile_end()
    print(f"{pr['merge_ms'] / pr['merge_launches'] * 1e3:.1f}")
    sys.exit(0)
for cfg, P in (("C3", 1), ("C3", 8), ("C2", 8)):
    res = []
    for w in ("1", "2", "4", "8"):
        r = subprocess.run([sys.executable, __file__, "--child", cfg, str(P)], capture_output=True, text=True,
                           env=dict(os.environ, TA_MERGE_W=w))
        res.append(f"W={w}: {r.stdout.strip() or r.stderr[-200:]} us")
    print(cfg, f"x{P}", " | ".join(res), flush=True)
