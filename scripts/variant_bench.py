"""Time C3 triangle (and optionally dense) for several library builds (TA_LIBRARY)."""
import glob, json, os, subprocess, sys
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
res = {}
for so in sorted(glob.glob(os.path.join(root, "variants", "lib_*.so"))):
    env = dict(os.environ, TA_LIBRARY=so)
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--no-cpu-baseline", "--no-e2e",
                          "--steps", "30"] + sys.argv[1:], env=env, capture_output=True, text=True)
    try:
        d = json.loads(out.stdout.strip().splitlines()[-1])
        res[os.path.basename(so)] = (round(d["ms_per_layer"], 4), round(d["value"], 1), d.get("dense_ms_per_layer"))
    except Exception as e:
        res[os.path.basename(so)] = ("ERR", out.stderr[-300:])
    print(os.path.basename(so), res[os.path.basename(so)], flush=True)
