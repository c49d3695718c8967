"""Per-instruction warp-stall breakdown from an ncu report (source page, SASS view)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]; data = rows[2:]
ix = {n: i for i, n in enumerate(h)}
stalls = [n for n in h if n.startswith("stall_") and "Not Issued" not in n]
S = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
tot = {s: sum(int(r[ix[s]] or 0) for r in data) for s in stalls}
print("kernel samples", S)
print("  ".join(f"{s[6:]}={v / S:.2f}" for s, v in sorted(tot.items(), key=lambda x: -x[1])[:10]))
order = sorted(range(len(data)), key=lambda i: -int(data[i][ix["Warp Stall Sampling (All Samples)"]] or 0))
for i in order[:top]:
    r = data[i]
    n = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    br = sorted(((int(r[ix[s]] or 0), s[6:]) for s in stalls), reverse=True)[:3]
    print(f"{i:5d} {n:6d} {r[1].strip()[:58]:58s} " + " ".join(f"{b}={a}" for a, b in br if a))
