"""Time C3 triangle (and dense) for several library builds (TA_LIBRARY), interleaved over
`--rounds` passes (box-to-box and run-to-run noise is ~2 %); reports the min per build."""
import glob, json, os, subprocess, sys
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
args = sys.argv[1:]
rounds = 2
if "--rounds" in args:
    i = args.index("--rounds"); rounds = int(args[i + 1]); del args[i:i + 2]
sos = sorted(glob.glob(os.path.join(root, "variants", "lib_*.so")))
res = {os.path.basename(s): [] for s in sos}
for r in range(rounds):
    for so in (sos if r % 2 == 0 else sos[::-1]):
        env = dict(os.environ, TA_LIBRARY=so)
        out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--no-cpu-baseline", "--no-e2e",
                              "--steps", "30"] + args, env=env, capture_output=True, text=True)
        try:
            d = json.loads(out.stdout.strip().splitlines()[-1])
            res[os.path.basename(so)].append((round(d["ms_per_layer"], 4), d.get("dense_ms_per_layer"),
                                              d.get("clocks", {}).get("sm_mhz"), round(d["kernel_ms"]["attn"], 4)))
        except Exception:
            res[os.path.basename(so)].append(("ERR", out.stderr[-300:]))
for k, v in res.items():
    ok = [x for x in v if x[0] != "ERR"]
    best = min(ok) if ok else v
    print(k, "min", best, "all", [(x[0], x[2]) if len(x) > 2 else x[0] for x in v], flush=True)
