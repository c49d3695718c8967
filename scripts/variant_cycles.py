"""Clock-independent comparison of kernel variants: for every variants/trace_*.so (TA_TRACE
builds) run the C3 triangle layer and report the median cycles per 5-block STREAM item and
per 128-block item of CTA 0 (SM clock varies with power draw; cycles do not)."""
import glob, os, subprocess, sys
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
for so in sorted(glob.glob(os.path.join(root, "variants", "trace_*.so"))):
    env = dict(os.environ, TA_LIBRARY=so)
    out = subprocess.run([sys.executable, os.path.join(root, "scripts", "trace_timeline.py"), cfg],
                         env=env, capture_output=True, text=True)
    lines = [l for l in out.stdout.splitlines() if l.startswith("items with")]
    print(os.path.basename(so), " | ".join(l.split(":", 1)[1].strip() for l in lines) or out.stderr[-300:],
          flush=True)
