"""Merge kernel time (library events) per build in variants/clk_*.so (e.g. TA_MERGE_U
variants) and warps-per-row setting (TA_MERGE_W), at C3 x1, C3 x8 and C2 x8 shard shapes."""
import glob
import os
import subprocess
import sys

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
child = os.path.join(root, "scripts", "merge_w.py")
for so in sorted(glob.glob(os.path.join(root, "variants", "clk_*.so"))):
    for cfg, P in (("C3", 1), ("C3", 8), ("C2", 8)):
        res = []
        for w in ("1", "4", "8"):
            r = subprocess.run([sys.executable, child, "--child", cfg, str(P)], capture_output=True, text=True,
                               env=dict(os.environ, TA_MERGE_W=w, TA_LIBRARY=so))
            res.append(f"W={w}: {r.stdout.strip() or r.stderr[-120:]}")
        print(os.path.basename(so), cfg, f"x{P}", " | ".join(res), flush=True)
