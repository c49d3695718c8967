#!/usr/bin/env python
"""bench.py -- TriangleMix prefill attention on B200 (driver contract, one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N ... bench.py --gpus N ...

Workload: BASELINE.json configs[2], one deep (triangle) layer of
Llama-3.1-8B attention (Hq=32, Hkv=8, d=128) at N=131072 tokens, si/sl/last =
8/512/128, bf16 synthetic iid N(0,1) Q/K/V (synth recipe).  At N GPUs
the layer is KV-head sharded (rank r owns kv heads [r*8/N, (r+1)*8/N) and their
q heads) and each step ends with the NCCL all-gather of O, so the
total work per step is fixed: "scaling": "strong".

A step = one pass of the hot path over the layer: the persistent attention kernel
(STREAM + LASTQ items), the LSE merge kernel, [the O all-gather].  value = kept-FLOP
TFLOP/s of the whole layer (4*d*Hq*kept pairs, closed form) / max-over-ranks step
time.  The dense causal layer (the speedup denominator) is timed in the same run.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402

L2_FLUSH_BYTES = 512 << 20
# One metric string for both arms (ours and --impl reference) so the driver can pair them.
METRIC = "triangle-attn prefill kept-FLOP TFLOP/s (ms/layer, speedup vs dense)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="C3", choices=sorted(synth.CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sweep", action="store_true", help="also time C2/C4a/C4b (extra JSON key)")
    ap.add_argument("--l2", choices=["flush", "inputs"], default="flush",
                    help="between timed steps: write a 512 MiB buffer (flush), or rely on the "
                         "inputs (1.5 GB at C3) exceeding the 126 MB L2 (inputs)")
    ap.add_argument("--gather", choices=["nccl", "fused", "multicast"], default="nccl",
                    help="N>1: O all-gather by NCCL after the kernel, or fused into the kernel "
                         "epilogue (f2: *_multi entry points storing into peer ranks' symmetric-"
                         "memory O buffers over NVLink; checked against NCCL once, falls back "
                         "to NCCL if the symmetric-memory rendezvous or the check fails), or fused "
                         "with multimem stores to the symmetric buffer's NVLS multicast address "
                         "(one egress per tile; same check and fallback)")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-points", action="store_true",
                    help="skip the C2 / Qwen 64K / Qwen 128K points and the shard-shape points")
    ap.add_argument("--dry-run", action="store_true",
                    help="launch plumbing only (no GPU): every rank joins a gloo group and rank 0 "
                         "prints the world it saw (tests the --gpus N self-spawn on CPU)")
    return ap.parse_args()


def config_dict(args, c, world, gather_mode=None):
    """The `config` object of the JSON line; identical in both arms (driver pairing)."""
    if gather_mode is None and world > 1:
        gather_mode = args.gather if args.gather == "nccl" else "fused"
    return {"workload": f"{args.workload}: {c.name}, one triangle (deep) layer, "
                        f"Hq={c.hq} Hkv={c.hkv} d={c.d} si/sl/last={c.si}/{c.sl}/{c.last}",
            "global_batch": 1, "seq_len": c.n,
            "parallelism": (f"kv-head shard x{world}" if world <= c.hkv else
                            f"q-head split x{world} ({world // c.hkv} ranks per kv head)")
                           + (f" + O all-gather: {gather_mode}" if world > 1 else ""),
            "l2": ("flushed (512 MiB write) before every timed step; inputs 1.5 GB > L2"
                   if args.l2 == "flush" else
                   "no flush: inputs (Q/K/V/O 1.5 GB at C3) exceed the 126 MB L2")}


def spawn_if_needed(args):
    """`python bench.py --gpus N` (N > 1) outside torchrun re-executes itself under
    torch.distributed.run with N ranks; under a launcher the world size must equal --gpus."""
    if "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
        if world != args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
        return
    if args.gpus <= 1:
        return
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def dry_run(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    ranks = [rank]
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        out = [None] * world
        dist.all_gather_object(out, rank)
        ranks = out
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"dry_run": True, "impl": args.impl, "n_gpus": world, "ranks": ranks,
                          "metric": METRIC}), flush=True)


# ------------------------------------------------------------------ helpers
def kept_flops(c, hq_local, dense=False):
    import paper_2507_21526_b200 as ta
    pairs = ta.pair_count(c.n, dense=True) if dense else ta.pair_count(c.n, c.si, c.sl, c.last)
    return 4 * c.d * hq_local * pairs


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return d.get("bf16_tflops"), d.get("bf16_tflops_sustained"), d.get("hbm_gbs"), "measured"
    return 1590.0, 1400.0, 6650.0, "fallback"


def ncu_traffic():
    """(dram bytes per launch, source label) of the attention kernel at C3 from the committed
    `ncu --set full` summary (dram__bytes_read.sum + dram__bytes_write.sum): DRAM counters
    are not readable from inside the timed run, so the capture is named with its round."""
    path = os.path.join(ROOT, "profiles", "ncu_attn_summary.json")
    if os.path.exists(path):
        try:
            d = json.load(open(path))
            return d.get("dram_bytes_per_launch"), d.get("source") or d.get("from")
        except Exception:
            return None, None
    return None, None


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons, pw = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            try:
                pw.append(float(f[2]))
            except ValueError:
                pass
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        loaded = [s for s in sm if s > 300] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w": statistics.median(pw) if pw else None}


def cpu_baseline_run(c, q, k, v, seconds, dense=False):
    """Time the fp64 C oracle on a bounded uniform row sample of the workload (all heads)."""
    import numpy as np

    from oracle import cref, masks  # noqa: F401  (bench's cpu_baseline leg only)
    cores = len(os.sched_getaffinity(0))

    def row_flops(rows):
        tot = 0
        for i in rows:
            i = int(i)
            if dense or i >= c.n - c.last:
                cnt = i + 1
            else:
                cnt = min(i + 1, c.si + c.sl)
            tot += cnt
        return 4 * c.d * c.hq * tot

    rng = np.random.default_rng(123)
    probe = np.sort(rng.choice(c.n, 4, replace=False))
    t0 = time.perf_counter()
    cref.attention(q, k, v, c.si, c.sl, c.last, dense, rows=probe, threads=cores)
    per_row = max((time.perf_counter() - t0) / len(probe), 1e-5)
    nrows = int(max(8, min(c.n, seconds / per_row)))
    rows = np.sort(rng.choice(c.n, nrows, replace=False))
    t0 = time.perf_counter()
    _, _, used = cref.attention(q, k, v, c.si, c.sl, c.last, dense, rows=rows, threads=cores)
    dt = time.perf_counter() - t0
    fl = row_flops(rows)
    fl_all = 4 * c.d * c.hq * (c.n * (c.n + 1) // 2 if dense else
                                cref.pair_count(c.n, c.si, c.sl, c.last, False))
    frac = fl / fl_all
    return {"value": fl / dt / 1e12, "unit": "TFLOP/s", "cores": int(used), "kind": "oracle",
            "sample": f"{nrows} uniformly sampled query rows x all {c.hq} q-heads of the "
                      f"{c.name} {'dense' if dense else 'triangle'} layer = {100 * frac:.1f} % of "
                      f"its kept pairs (fp64 C oracle, {dt:.1f} s wall; whole layer extrapolated "
                      f"{dt / frac:.0f} s)",
            "sampled_fraction": frac, "layer_seconds_extrapolated": dt / frac,
            "seconds": dt}


def cpu_extra_points(cores):
    """SURVEY 8(d) oracle timing beside the GPU numbers: C1 triangle and dense in full, C2
    dense on a bounded row sample (extrapolated by pair count, labelled)."""
    import numpy as np

    from oracle import cref
    out = []
    c1 = synth.CONFIGS["C1"]
    q, k, v = synth.config_qkv(c1)
    for dense in (False, True):
        t0 = time.perf_counter()
        cref.attention(q, k, v, c1.si, c1.sl, c1.last, dense, threads=1)
        dt = time.perf_counter() - t0
        pairs = c1.n * (c1.n + 1) // 2 if dense else cref.pair_count(c1.n, c1.si, c1.sl, c1.last, False)
        out.append({"workload": f"C1 {'dense' if dense else 'triangle'} (full)", "seconds": dt,
                    "cores": 1, "mpair_per_s": pairs * c1.hq / dt / 1e6})
    c2 = synth.CONFIGS["C2"]
    q, k, v = synth.config_qkv(c2, layer=0)
    rows = np.sort(np.random.default_rng(7).choice(c2.n, 64, replace=False))
    t0 = time.perf_counter()
    _, _, used = cref.attention(q, k, v, 0, 1, 1, True, rows=rows, threads=cores)
    dt = time.perf_counter() - t0
    sp = int(sum(int(i) + 1 for i in rows))
    allp = c2.n * (c2.n + 1) // 2
    out.append({"workload": "C2 dense (64 uniform rows, all heads; extrapolated by pair count)",
                "seconds": dt, "cores": int(used), "mpair_per_s": sp * c2.hq / dt / 1e6,
                "layer_seconds_extrapolated": dt * allp / sp})
    return out


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    c = synth.CONFIGS[args.workload]
    q, k, v = synth.config_qkv(c, layer=16)
    per_step = max(1.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    vals = []
    for s in range(args.warmup + args.steps):
        r = cpu_baseline_run(c, q, k, v, per_step)
        if s >= args.warmup:
            vals.append(r)
    tot_fl = sum(x["value"] * x["seconds"] for x in vals)
    tot_s = sum(x["seconds"] for x in vals)
    value = tot_fl / tot_s
    line = {
        "impl": "reference", "metric": METRIC,
        "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * tot_s / len(vals), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args, c, args.gpus),
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": vals[0]["cores"],
                         "kind": "oracle", "sample": vals[0]["sample"]},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def main():
    args = parse()
    if args.warmup < 3:
        args.warmup = 3
    spawn_if_needed(args)
    if args.dry_run:
        return dry_run(args)
    if args.impl == "reference":
        return run_reference(args)
    import paper_2507_21526_b200 as ta

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # Plumbing check on a 1-GPU box only (never for measurements): every rank on cuda:0,
    # gloo instead of NCCL (NCCL refuses two ranks on one GPU).
    one_gpu_check = os.environ.get("TA_BENCH_ONE_GPU_CHECK") == "1"
    if one_gpu_check:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if one_gpu_check:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    from paper_2507_21526_b200 import shard
    c = synth.CONFIGS[args.workload]
    try:
        plan = shard.head_plan(c.hq, c.hkv, world)   # kv-head shards, or q-head split (Qwen x8)
    except ValueError as e:
        raise SystemExit(str(e))
    hq_l = plan[rank][3] - plan[rank][2]
    q, k, v = synth.config_qkv(c, layer=16)      # CPU bf16, same recipe as the parity tests
    qs, ks, vs = (t.contiguous() for t in shard.shard_qkv(q, k, v, rank, world))
    qd, kd, vd = qs.to(dev), ks.to(dev), vs.to(dev)
    od = torch.empty_like(qd)
    o_full = torch.empty((c.hq, c.n, c.d), dtype=torch.bfloat16, device=dev) if world > 1 else None
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def layer_nccl(dense=False):
        if dense:
            ta.dense_attn_prefill(qd, kd, vd, od)
        else:
            ta.triangle_attn_prefill(qd, kd, vd, od, sink=c.si, window=c.sl, last_q=c.last)
        if world > 1:
            shard.gather_heads(od, world, out=o_full, plan=plan)

    layer = layer_nccl
    gather_mode = "nccl" if world > 1 else None
    o_result = od   # the buffer holding this rank's O after a step (e2e reads it back)
    if world > 1 and args.gather in ("fused", "multicast"):
        # f2: every rank's epilogue stores its O tiles into all ranks' symmetric-memory
        # full-O buffers (own slice + the same head slice of each peer); a device-side
        # barrier orders them before the next layer reads.  Verified once against NCCL.
        try:
            import torch.distributed._symmetric_memory as symm
            o_sym = symm.empty((c.hq, c.n, c.d), dtype=torch.bfloat16, device=dev)
            hdl = symm.rendezvous(o_sym, dist.group.WORLD)
            h0, h1 = plan[rank][2], plan[rank][3]
            peers = [hdl.get_buffer(r, (c.hq, c.n, c.d), torch.bfloat16)[h0:h1]
                     for r in range(world) if r != rank]
            own = o_sym[h0:h1]
            mc_ptr = int(getattr(hdl, "multicast_ptr", 0) or 0) if args.gather == "multicast" else 0
            if args.gather == "multicast" and not mc_ptr:
                raise RuntimeError("symmetric memory has no multicast (NVLS) address on this box")
            mc_slice = mc_ptr + h0 * c.n * c.d * 2   # this rank's heads inside the full O

            def layer_fused(dense=False):
                if mc_ptr:   # one multimem store per tile; the NVSwitch replicates it
                    if dense:
                        ta.dense_attn_prefill_multicast(qd, kd, vd, mc_slice, (c.n * c.d, c.d), own)
                    else:
                        ta.triangle_attn_prefill_multicast(qd, kd, vd, mc_slice, (c.n * c.d, c.d),
                                                           own, sink=c.si, window=c.sl,
                                                           last_q=c.last)
                elif dense:
                    ta.dense_attn_prefill_multi(qd, kd, vd, peers, own)
                else:
                    ta.triangle_attn_prefill_multi(qd, kd, vd, peers, own, sink=c.si, window=c.sl,
                                                   last_q=c.last)
                hdl.barrier(channel=0)

            layer_nccl()
            layer_fused()
            torch.cuda.synchronize()
            ok = torch.tensor([1.0 if torch.equal(o_sym, o_full) else 0.0], device=dev)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if ok.item() == 1.0:
                layer, gather_mode = layer_fused, ("fused multicast (kernel epilogue multimem stores "
                                                   "-> NVLS)" if mc_ptr else
                                                   "fused (kernel epilogue -> peer symmetric memory)")
                o_result = own
            else:
                gather_mode = "nccl (fused output check failed)"
        except Exception as e:  # no P2P / symmetric memory on this box: report and keep NCCL
            gather_mode = f"nccl (fused unavailable: {type(e).__name__}: {str(e)[:120]})"

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            if one_gpu_check:
                dist.barrier()
            else:
                dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    def timed(steps, dense=False, profile=False):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(steps)]
        barrier()
        if profile:
            ta.profile_begin()
        for s in range(steps):
            if args.l2 == "flush":
                flush.zero_()             # L2 flush between timed iterations (> 126 MB L2)
            evs[s][0].record(stream)
            layer(dense)
            evs[s][1].record(stream)
        barrier()
        prof = ta.profile_end() if profile else None
        ms = sum(a.elapsed_time(b) for a, b in evs)
        return max_over_ranks(ms / steps), prof

    # ---- triangle layer: warmup + timed
    for _ in range(args.warmup):
        layer()
    sampler = ClockSampler(local)
    sampler.start()
    ms_tri, prof = timed(args.steps, profile=True)
    attn_ms = max_over_ranks(prof["attn_ms"] / max(1, prof["attn_launches"]))
    merge_ms = max_over_ranks(prof["merge_ms"] / max(1, prof["merge_launches"]))
    gpu_launches = prof["attn_launches"] + prof["merge_launches"]

    # ---- PDL: the same step with the merge launched without programmatic dependent launch
    # (outer events only, no per-kernel events between the two launches)
    pdl = None
    if world == 1 and not args.no_points:
        def step_ms(n):
            evs = []
            barrier()
            for _ in range(n):
                if args.l2 == "flush":
                    flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                layer()
                b.record(stream)
                evs.append((a, b))
            barrier()
            return statistics.median(a.elapsed_time(b) for a, b in evs)
        on, off = [], []
        for r in range(8):   # ABBA order: clock drift under the power cap cancels
            pdl_on = r % 4 in (0, 3)
            ta.set_pdl(pdl_on)
            (on if pdl_on else off).append(step_ms(10))
        ta.set_pdl(True)
        pdl = {"step_ms_pdl": statistics.median(on), "step_ms_no_pdl": statistics.median(off),
               "saved_us": 1e3 * (statistics.median(off) - statistics.median(on)),
               "what": "median step (attention + merge) with the merge launched with / without "
                       "programmatic dependent launch, 4 + 4 runs of 10 steps in ABBA order"}

    fl_layer = kept_flops(c, c.hq)
    fl_rank = kept_flops(c, hq_l)
    value = fl_layer / (ms_tri * 1e-3) / 1e12

    # ---- dense layer (speedup denominator), same shard
    dense_ms = None
    if not args.no_dense:
        layer(dense=True)
        dense_ms, _ = timed(3, dense=True)
    clocks = sampler.stop()   # sampled over the triangle and dense timed regions

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e and world == 1:
        # End to end through the public API with host buffers, pipelined two deep across
        # steps: step i's H2D (copy stream) and step i-1's D2H (second copy stream) overlap
        # step i-1 / i's kernels; every step still copies its own Q/K/V in from pinned host
        # memory and its O back out inside the timed region.
        qh, kh, vh = qs.pin_memory(), ks.pin_memory(), vs.pin_memory()
        sets = [(qd, kd, vd, od), tuple(torch.empty_like(t) for t in (qd, kd, vd, od))]
        ohs = [torch.empty(od.shape, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        e_steps = max(4, min(args.steps, 8))
        ev = lambda: torch.cuda.Event()  # noqa: E731
        done = [None, None]      # kernel of the set finished (inputs free, O ready)
        drained = [None, None]   # D2H of the set's O finished

        def e2e_run(n):
            for i in range(n):
                sset = i % 2
                q_, k_, v_, o_ = sets[sset]
                with torch.cuda.stream(s_in):
                    if done[sset] is not None:
                        s_in.wait_event(done[sset])
                    q_.copy_(qh, non_blocking=True)
                    k_.copy_(kh, non_blocking=True)
                    v_.copy_(vh, non_blocking=True)
                    e_in = ev()
                    e_in.record(s_in)
                stream.wait_event(e_in)
                if drained[sset] is not None:
                    stream.wait_event(drained[sset])
                ta.triangle_attn_prefill(q_, k_, v_, o_, sink=c.si, window=c.sl, last_q=c.last,
                                         stream=stream)
                done[sset] = ev()
                done[sset].record(stream)
                with torch.cuda.stream(s_out):
                    s_out.wait_event(done[sset])
                    ohs[sset].copy_(o_, non_blocking=True)
                    drained[sset] = ev()
                    drained[sset].record(s_out)

        e2e_run(2)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        s_in.wait_stream(stream)
        e2e_run(e_steps)
        s_out.synchronize()
        stream.wait_stream(s_out)
        e1.record(stream)
        barrier()
        e_ms = e0.elapsed_time(e1) / e_steps
        e2e = {"value": fl_layer / (e_ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": e_ms,
               "h2d_bytes_per_step": int((qh.numel() + kh.numel() + vh.numel()) * 2),
               "d2h_bytes_per_step": int(ohs[0].numel() * 2), "steps": e_steps,
               "overlap": "2-deep pipeline over steps: H2D on a copy stream | kernels | D2H on a "
                          "second copy stream (PCIe-bound)"}
        del sets
    elif not args.no_e2e:
        qh, kh, vh = qs.pin_memory(), ks.pin_memory(), vs.pin_memory()
        oh = torch.empty(o_result.shape, dtype=torch.bfloat16).pin_memory()
        e_steps = min(args.steps, 3)

        def e2e_step():
            qd.copy_(qh, non_blocking=True)
            kd.copy_(kh, non_blocking=True)
            vd.copy_(vh, non_blocking=True)
            layer()
            oh.copy_(o_result, non_blocking=True)

        e2e_step()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(e_steps):
            e2e_step()
        e1.record(stream)
        barrier()
        e_ms = max_over_ranks(e0.elapsed_time(e1) / e_steps)
        e2e = {"value": fl_layer / (e_ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": e_ms,
               "h2d_bytes_per_step": int((qh.numel() + kh.numel() + vh.numel()) * 2),
               "d2h_bytes_per_step": int(oh.numel() * 2)}

    # ---- sweep of the other configs (1 GPU only; extra key)
    sweep = None
    if not args.no_points and world == 1:
        sweep = []
        for name in ("C2", "C4a", "C4b"):
            cc = synth.CONFIGS[name]
            q2, k2, v2 = (t.to(dev) for t in synth.config_qkv(cc, layer=cc.tri_start))
            o2 = torch.empty_like(q2)
            res = {}
            for dn in (False, True):
                fn = (lambda: ta.dense_attn_prefill(q2, k2, v2, o2)) if dn else (
                    lambda: ta.triangle_attn_prefill(q2, k2, v2, o2, sink=cc.si, window=cc.sl,
                                                     last_q=cc.last))
                for _ in range(3):
                    fn()
                reps = 3 if dn else 10
                evs = []
                barrier()
                for _ in range(reps):
                    flush.zero_()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    fn()
                    b.record(stream)
                    evs.append((a, b))
                barrier()
                res["dense_ms" if dn else "triangle_ms"] = sum(a.elapsed_time(b) for a, b in evs) / reps
            res["triangle_tflops"] = kept_flops(cc, cc.hq) / (res["triangle_ms"] * 1e-3) / 1e12
            res["dense_tflops"] = kept_flops(cc, cc.hq, True) / (res["dense_ms"] * 1e-3) / 1e12
            res["speedup_vs_dense"] = res["dense_ms"] / res["triangle_ms"]
            res["workload"] = cc.name
            sweep.append(res)
            del q2, k2, v2, o2

    # ---- strong-scaling proxy on 1 GPU: the per-rank kernel at the 2/4/8-way kv-head
    # shard shapes of C3, C2 and Qwen 128K; efficiency = (full-layer ms / P) / shard ms.
    shard_pts = None
    if not args.no_points and world == 1:
        shard_pts = []
        for name in ("C3", "C2", "C4b"):   # Llama 128K / 32K, Qwen2.5-7B 128K
            cc = synth.CONFIGS[name]
            full = None
            for P in (1, 2, 4, 8):
                # per-rank shapes of shard.head_plan (kv-head shards; Qwen at 8 ranks splits
                # each kv head's 7 q heads 3 + 4): time each distinct shape, the step is the max
                shapes = sorted({(q1_ - q0_, kv1_ - kv0_) for kv0_, kv1_, q0_, q1_ in
                                 shard.head_plan(cc.hq, cc.hkv, P)})
                kms = 0.0
                for hq_r, hkv_r in shapes:
                    q1, k1, v1 = (t.to(dev) for t in synth.make_qkv(hq_r, hkv_r, cc.n, cc.d, seed=100 + P))
                    o1 = torch.empty_like(q1)
                    fn = lambda: ta.triangle_attn_prefill(q1, k1, v1, o1, sink=cc.si, window=cc.sl,
                                                          last_q=cc.last)
                    for _ in range(3):
                        fn()
                    barrier()
                    ta.profile_begin()
                    for _ in range(10):
                        flush.zero_()
                        fn()
                    barrier()
                    pr = ta.profile_end()
                    kms = max(kms, (pr["attn_ms"] + pr["merge_ms"]) / 10)
                    del q1, k1, v1, o1
                if P == 1:
                    full = kms
                shard_pts.append({"workload": name, "ranks": P,
                                  "hq_per_rank": "/".join(str(h) for h, _ in shapes),
                                  "kernel_ms_per_rank": kms,
                                  "strong_scaling_eff": full / (P * kms)})

    # ---- NEXT rows on 1 GPU (extra keys): final-layer last rows (f1), StreamingMix (f3),
    # and the C5 attention stack per rank of an 8-way kv-head shard (16 dense + 16 triangle).
    extras = None
    if args.sweep and world == 1:
        extras = {}

        def dev_ms(fn, reps):
            for _ in range(2):
                fn()
            evs = []
            barrier()
            for _ in range(reps):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                fn()
                b.record(stream)
                evs.append((a, b))
            barrier()
            return sum(a.elapsed_time(b) for a, b in evs) / reps

        r = c.last
        o_last = torch.empty((c.hq, r, c.d), dtype=torch.bfloat16, device=dev)
        ms = dev_ms(lambda: ta.last_rows_attn_prefill(qd, kd, vd, o_last, last_q=r), 10)
        fl = 4 * c.d * c.hq * sum(range(c.n - r + 1, c.n + 1))
        extras["final_layer_last_rows"] = {
            "what": f"{c.name}: last {r} rows over all causal keys (P:L245-247)", "ms": ms,
            "kept_tflops": fl / (ms * 1e-3) / 1e12}
        ms = dev_ms(lambda: ta.triangle_attn_prefill(qd, kd, vd, od, sink=c.si, window=c.sl, last_q=0), 10)
        fl = 4 * c.d * c.hq * ta.pair_count(c.n, c.si, c.sl, 0)
        extras["streamingmix_layer"] = {"what": f"{c.name}: sink {c.si} + window {c.sl}, last 0",
                                        "ms": ms, "kept_tflops": fl / (ms * 1e-3) / 1e12}
        stack = []
        g8 = c.hq // c.hkv
        for n in (32768, 65536, 131072):
            q1, k1, v1 = (t.to(dev) for t in synth.make_qkv(g8, 1, n, c.d, seed=n))
            o1 = torch.empty_like(q1)
            tri = dev_ms(lambda: ta.triangle_attn_prefill(q1, k1, v1, o1, sink=c.si, window=c.sl,
                                                          last_q=c.last), 5)
            den = dev_ms(lambda: ta.dense_attn_prefill(q1, k1, v1, o1), 2)
            stack.append({"seq_len": n, "triangle_ms": tri, "dense_ms": den,
                          "stack_ms_16d_16t": 16 * den + 16 * tri, "stack_ms_32d": 32 * den,
                          "attention_speedup": (32 * den) / (16 * den + 16 * tri)})
            del q1, k1, v1, o1
        extras["c5_stack_per_rank_of_8"] = {
            "what": "per-rank attention kernels of the 32-layer Llama stack (16 dense + 16 triangle, "
                    "tri_start=16) at an 8-way kv-head shard (1 kv head, 4 q heads per rank); "
                    "all-gather not included; 1 GPU measures one rank", "points": stack}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_run(c, q, k, v, args.cpu_seconds)
        cpu.pop("seconds", None)
        cpu["extra_points"] = cpu_extra_points(cpu["cores"])

    if rank == 0:
        peak, peak_sus, hbm, src = measured_peaks()
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        achieved = fl_rank / (attn_ms * 1e-3) / 1e12
        traffic, traffic_src = ncu_traffic() if (args.workload == "C3" and world == 1) else (None, None)
        # compulsory bytes of the layer shard: bf16 Q, O (hq_l heads) and K, V (kv heads)
        hkv_l = plan[rank][1] - plan[rank][0]
        alg_bytes = 2 * c.n * c.d * (2 * hq_l + 2 * hkv_l)
        hbm_line = {"algorithmic_bytes_per_launch": alg_bytes,
                    "algorithmic_gbs": alg_bytes / (attn_ms * 1e-3) / 1e9,
                    "dram_bytes_per_launch": traffic,
                    "dram_gbs": (traffic / (attn_ms * 1e-3) / 1e9) if traffic else None,
                    "peak_gbs": hbm,
                    "dram_source": traffic_src,
                    "note": "dram bytes from the ncu --set full capture named in dram_source, "
                            "divided by this run's CUDA-event kernel time"}
        line = {
            "metric": METRIC,
            "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_tri, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded iid N(0,1) bf16 Q/K/V, synth recipe)",
            "config": config_dict(args, c, world, gather_mode),
            "ms_per_layer": ms_tri,
            "dense_ms_per_layer": dense_ms,
            "speedup_vs_dense": (dense_ms / ms_tri) if dense_ms else None,
            "dense_tflops": (kept_flops(c, c.hq, True) / (dense_ms * 1e-3) / 1e12) if dense_ms else None,
            "dense_frac_of_peak": ((kept_flops(c, c.hq, True) / (dense_ms * 1e-3) / 1e12) / peak
                                   if dense_ms else None),
            "kernel_ms": {"attn": attn_ms, "merge": merge_ms},
            # N > 1: the rest of the step is the O all-gather (NCCL, or the fused f2 barrier)
            "gather_ms": (max(0.0, ms_tri - attn_ms - merge_ms) if world > 1 else None),
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "peak_source": f"{src} bf16 burst (MEASURED_PEAKS.json)",
                         "kernel": "attn_kernel<128> (persistent tcgen05 flash attention)",
                         "algorithmic_flops_per_launch": fl_rank,
                         # the same achieved FLOP/s against the dense bf16 tensor rate at the SM
                         # clock sampled during this run (148 SMs x 8192 FLOP/clk): how much of
                         # the gap to `peak` is the power-capped clock rather than the kernel
                         "peak_at_run_clock": (sms * 8192 * clocks["sm_mhz"] * 1e6 / 1e12
                                               if clocks.get("sm_mhz") else None),
                         "frac_at_run_clock": (achieved / (sms * 8192 * clocks["sm_mhz"] * 1e6 / 1e12)
                                               if clocks.get("sm_mhz") else None)},
            "hbm": hbm_line,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": gpu_launches,
            "clocks": clocks,
            "paper_context": "A100 Triton triangle 12/24/49 ms (3.7x/7.5x/15.3x vs FlashAttention) "
                             "at 32K/64K/128K, P:L433-436; other hardware, context only",
        }
        if sweep is not None:
            line["points"] = sweep
        if shard_pts is not None:
            line["shard_points"] = shard_pts
        if pdl is not None:
            line["pdl"] = pdl
        if extras is not None:
            line["next_rows"] = extras
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
