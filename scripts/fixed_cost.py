"""Per-launch fixed cost of the attention path: kernel time (library events) for tiny problems
(one item per CTA or less), triangle and dense, plus the empty-ish launch gap."""
import os
import sys

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, root)
import torch  # noqa: E402

import paper_2507_21526_b200 as ta  # noqa: E402
import synth  # noqa: E402

for (hq, hkv, n) in [(1, 1, 64), (4, 1, 64), (4, 1, 4096), (4, 1, 9472), (32, 8, 4096)]:
    q, k, v = (t.cuda() for t in synth.make_qkv(hq, hkv, n, 128, seed=1))
    for dense in (False, True):
        fn = (lambda: ta.dense_attn_prefill(q, k, v)) if dense else (lambda: ta.triangle_attn_prefill(q, k, v))
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        ta.profile_begin()
        for _ in range(50):
            fn()
        torch.cuda.synchronize()
        pr = ta.profile_end()
        a = pr["attn_ms"] / max(1, pr["attn_launches"]) * 1e3
        m = pr["merge_ms"] / max(1, pr["merge_launches"]) * 1e3 if pr["merge_launches"] else 0
        print(f"hq{hq} hkv{hkv} n{n} {'dense' if dense else 'tri'}: attn {a:.1f} us, merge {m:.1f} us", flush=True)
