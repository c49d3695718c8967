"""Build TA_CTA_CLOCK kernel variants for scripts/variant_ctaclk.py.

    python scripts/build_variants.py NAME=DEF1,DEF2 NAME2=DEF3 ...
    python scripts/build_variants.py base= sumr3=TA_SUM_ROUNDED=3

Each variant lands in variants/clk_<NAME>.so (git-ignored; travels with gpurun).  The
builds run in parallel."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, root)
from paper_2507_21526_b200 import build as b  # noqa: E402

os.makedirs(os.path.join(root, "variants"), exist_ok=True)
jobs = []
for arg in sys.argv[1:]:
    name, _, defs = arg.partition("=")
    defines = ["TA_CTA_CLOCK"] + [d for d in defs.split(",") if d]
    jobs.append((name, defines))


def one(job):
    name, defines = job
    out = os.path.join(root, "variants", f"clk_{name}.so")
    b.build(force=True, defines=defines, out=out)
    return out


with ThreadPoolExecutor(max_workers=8) as ex:
    for out in ex.map(one, jobs):
        print(out)
