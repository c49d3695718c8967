"""Sustained power-capped A/B of kernel builds: each variants/clk_*.so runs C3 triangle
back to back for a few seconds (no L2 flush) while nvidia-smi samples power and SM clock;
reports ms per call, W and MHz (medians), interleaved over rounds.  Under the board power
cap the SM clock follows the power a kernel draws, so this is the metric a sustained run
sees (the 20-step bench is too short to reach it)."""
import glob
import json
import os
import statistics
import subprocess
import sys
import threading
import time

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, root)
    import torch
    import paper_2507_21526_b200 as ta
    secs = float(sys.argv[2])
    g = torch.Generator(device="cuda").manual_seed(1)
    n, hq, hkv = 131072, 32, 8
    q = torch.randn(hq, n, 128, device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn(hkv, n, 128, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(hkv, n, 128, device="cuda", generator=g).to(torch.bfloat16)
    o = torch.empty_like(q)
    fn = lambda: ta.triangle_attn_prefill(q, k, v, o, sink=8, window=512, last_q=128)  # noqa: E731
    for _ in range(200):
        fn()
    torch.cuda.synchronize()
    lines = []
    smi = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=power.draw,clocks.sm",
                            "--format=csv,noheader,nounits", "-lms", "100"],
                           stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
    th = threading.Thread(target=lambda: [lines.append(ln) for ln in smi.stdout], daemon=True)
    th.start()
    ms = []
    t_end = time.time() + secs
    while time.time() < t_end:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(50):
            fn()
        b.record()
        b.synchronize()
        ms.append(a.elapsed_time(b) / 50)
    smi.terminate()
    pw, mhz = [], []
    for ln in lines:
        try:
            p_, c_ = (float(x) for x in ln.split(","))
            pw.append(p_)
            mhz.append(c_)
        except ValueError:
            pass
    print(json.dumps({"ms": statistics.median(ms), "W": statistics.median(pw) if pw else None,
                      "MHz": statistics.median(mhz) if mhz else None}))
    sys.exit(0)
sos = sorted(glob.glob(os.path.join(root, "variants", "clk_*.so")))
secs = os.environ.get("SECS", "4")
res = {os.path.basename(s): [] for s in sos}
for rnd in range(int(os.environ.get("ROUNDS", "2"))):
    for so in (sos if rnd % 2 == 0 else sos[::-1]):
        r = subprocess.run([sys.executable, __file__, "--child", secs], env=dict(os.environ, TA_LIBRARY=so),
                           capture_output=True, text=True)
        try:
            res[os.path.basename(so)].append(json.loads(r.stdout.strip().splitlines()[-1]))
        except Exception:
            res[os.path.basename(so)].append(r.stderr[-300:])
for k_, v_ in res.items():
    print(k_, v_, flush=True)
