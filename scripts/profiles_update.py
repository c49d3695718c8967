"""Copy a gpu_final.sh run from gpurun_out/ into profiles/ (bench lines, launch list +
summary, ncu full summary + stall breakdown, memcheck, pytest/smoke, TTFT).

    python scripts/profiles_update.py r01
"""
import csv, os, shutil, statistics, subprocess, sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(root, "gpurun_out"), os.path.join(root, "profiles")
rows = list(csv.reader(open(os.path.join(G, f"launches_{tag}.csv"))))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
ls = [(r[ki], float(r[vi].replace(",", "")) / 1000) for r in rows[hi + 1:]
      if len(r) > vi and r[mi] == "gpu__time_duration.sum"]
out = ["ncu --metrics gpu__time_duration.sum --clock-control none --csv (launch list of: "
       "python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-points)",
       "cold-cache, serialised per-launch times: compare shares, not absolutes.", "",
       "per launch (us), in order:"]
out += [f"  {n[:48]:48s} {t:10.1f}" for n, t in ls]
tri = [t for n, t in ls if "attn_kernel" in n and t < 5000]
mer = [t for n, t in ls if "merge" in n]
a, m = statistics.median(tri), statistics.median(mer)
out += ["", f"triangle step under ncu: attn_kernel {a:.1f} us + merge {m:.1f} us -> "
        f"attn share {100 * a / (a + m):.1f}% of the step"]
open(os.path.join(P, f"{tag}_launches_summary.txt"), "w").write("\n".join(out) + "\n")
shutil.copy(os.path.join(G, f"launches_{tag}.csv"), os.path.join(P, f"{tag}_launches.csv"))
shutil.copy(os.path.join(G, f"memcheck_{tag}.log"), os.path.join(P, f"{tag}_memcheck.log"))
shutil.copy(os.path.join(G, f"ttft_{tag}.json"), os.path.join(P, f"{tag}_ttft.json"))
for src, dst in ((f"bench_{tag}.json", f"{tag}_bench.json"), (f"bench_ref_{tag}.json", f"{tag}_bench_reference.json")):
    line = open(os.path.join(G, src)).read().strip().splitlines()[-1]
    open(os.path.join(P, dst), "w").write(line + "\n")
with open(os.path.join(P, f"{tag}_pytest_gpu.txt"), "w") as f:
    f.write(open(os.path.join(G, f"pytest_gpu_{tag}.log")).read().strip().splitlines()[-1] + "\n")
    f.write("smoke: " + open(os.path.join(G, f"smoke_{tag}.log")).read().strip().splitlines()[-1] + "\n")
rep = os.path.join(G, f"prof_attn_{tag}.ncu-rep")
subprocess.run([sys.executable, os.path.join(root, "scripts", "ncu_summary.py"), rep, tag], check=True,
               capture_output=True)
with open(os.path.join(P, f"{tag}_ncu_stalls.txt"), "w") as f:
    subprocess.run([sys.executable, os.path.join(root, "scripts", "ncu_stalls.py"), rep], stdout=f, check=True)
print("\n".join(out[-1:]))
