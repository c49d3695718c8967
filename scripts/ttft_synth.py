"""Synthetic-weight TTFT of a Llama-3.1-8B-shaped prefill (structure of
the paper's tab:efficiency_ttft): all-dense attention vs TriangleMix
(16 dense + 16 triangle layers), plus the final-layer last-rows mode.  Random weights,
synthetic inputs; GEMMs via cuBLAS, attention via libtriattn.  One JSON line."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_21526_b200 import prefill_model as pm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ns", default="32768,49152,65536,81920,98304,114688,131072")
ap.add_argument("--model", default="llama", choices=["llama", "qwen"])
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
dev = torch.device("cuda")
shape = pm.LLAMA31_8B if args.model == "llama" else pm.QWEN25_7B
m = pm.SyntheticPrefill(shape, dev)
out = {"model": shape.name + " (random weights, shapes only)", "tri_start": shape.tri_start,
       "si/sl/last": [8, 512, 128], "unit": "s", "points": []}
for n in [int(x) for x in args.ns.split(",")]:
    x = (torch.randn(n, shape.hidden, device=dev) * 0.5).to(torch.bfloat16)
    res = {"seq_len": n}
    for label, mode, flr in (("dense", "dense", False), ("trianglemix", "trianglemix", False),
                             ("trianglemix_final_last_rows", "trianglemix", True)):
        m.forward(x[:4096], mode=mode, final_last_rows=flr)  # warm-up (kernels, schedules)
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            y = m.forward(x, mode=mode, final_last_rows=flr)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) / 1e3)
        res[label] = min(ts)
        res[label + "_finite"] = bool(torch.isfinite(y.float()).all().item())
    res["trianglemix_vs_dense"] = res["trianglemix"] / res["dense"] - 1.0
    out["points"].append(res)
    print(json.dumps(res), file=sys.stderr, flush=True)
    del x
print(json.dumps(out))
