"""Summarise an ncu --set full capture of attn_kernel into profiles/ (json + text).

    python scripts/ncu_summary.py gpurun_out/prof_attn_r01.ncu-rep r01
"""
import csv, io, json, os, subprocess, sys

rep, tag = sys.argv[1], sys.argv[2]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
m = {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def num(key, scale=1.0):
    v, u = m[key]
    x = float(v.replace(",", ""))
    mult = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1e-3, "us": 1e-6, "ns": 1e-9}.get(u, 1)
    return x * mult * scale


want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_srcunit_tex_lookup_hit.sum", "lts__t_sectors_srcunit_tex_lookup_miss.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "gpc__cycles_elapsed.max"]
out = {}
for k in want:
    if k in m:
        out[k] = m[k][0] + (" " + m[k][1] if m[k][1] else "")
dram = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
dur = num("gpu__time_duration.sum")
summary = {"tag": tag, "kernel": "attn_kernel<128>", "source": os.path.basename(rep),
           "command": "ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 3 -c 1 "
                      "python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-dense --no-e2e --no-points",
           "dram_bytes_per_launch": dram, "duration_s_under_ncu": dur, "metrics": out}
os.makedirs(os.path.join(root, "profiles"), exist_ok=True)
json.dump(summary, open(os.path.join(root, "profiles", f"{tag}_ncu_attn_full.json"), "w"), indent=1)
json.dump({"dram_bytes_per_launch": dram, "source": f"profiles/{tag}_ncu_attn_full.json (ncu --set full, round {tag})"},
          open(os.path.join(root, "profiles", "ncu_attn_summary.json"), "w"), indent=1)
print(json.dumps(summary, indent=1))
