"""Build libtriattn.so in-tree with nvcc for sm_100a (no torch extension machinery).

    python -m paper_2507_21526_b200.build [--verbose]

The .so lands next to this file so it travels to the GPU box with the repo
snapshot (it is git-ignored).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libtriattn.so")
SO_TRACE = os.path.join(HERE, "libtriattn_trace.so")
SO_COUNT = os.path.join(HERE, "libtriattn_count.so")  # TA_COUNT: per-row pair counters
SOURCES = ["api.cu", "kernels.cu", "schedule.cpp"]
HEADERS = ["ptx.cuh", "kernel_params.h", "schedule.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "triattn.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def _stale_so(so: str) -> bool:
    if not os.path.exists(so):
        return True
    t = os.path.getmtime(so)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "triattn.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def build_count(force: bool = False) -> str:
    """The TA_COUNT build (libtriattn_count.so): same kernels, plus per-row counters of the
    admitted pairs and computed S columns (GPU-side kept-work proof, tests/test_gpu_count.py)."""
    if not force and not _stale_so(SO_COUNT):
        return SO_COUNT
    return build(force=True, defines=("TA_COUNT",), out=SO_COUNT)


def build(force: bool = False, verbose: bool = False, trace: bool = False, defines=(),
          out: str | None = None) -> str:
    """Compile libtriattn.so (or, with trace=True, the debug-timeline libtriattn_trace.so;
    `defines`/`out` build tuning variants for experiments)."""
    so = out or (SO_TRACE if trace else SO)
    if not force and not trace and out is None and not _stale():
        return SO
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
           "--expt-relaxed-constexpr",
           "-I" + os.path.join(os.path.dirname(HERE), "include"),
           "-o", so + ".tmp"] + [os.path.join(CSRC, f) for f in SOURCES]
    if trace:
        cmd.insert(1, "-DTA_TRACE")
    for d in defines:
        cmd.insert(1, "-D" + d)
    cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise subprocess.CalledProcessError(r.returncode, cmd)
    if verbose:
        sys.stderr.write(r.stderr)
    spills = _attn_spills(r.stderr)
    hot = [x for x in spills if "attn_kernelILi128ELi0E" in x]
    if hot and so == SO:
        # A spill in the hot instantiation put local-memory loads on the MMA issue path
        # (measured: tcgen05.mma groups waited on an LDL of the TMEM base); refuse it.
        raise RuntimeError("attn_kernel<128, single output> spills registers: " + "; ".join(hot))
    for x in spills:
        if x not in hot:
            sys.stderr.write("warning: " + x + "\n")
    os.replace(so + ".tmp", so)
    return so


def _attn_spills(ptxas_log: str):
    """ptxas -v lines reporting spills for the attention kernel instantiations."""
    out, cur = [], None
    for ln in ptxas_log.splitlines():
        if "Function properties for" in ln:
            cur = ln.split("for", 1)[1].strip()
        elif "spill" in ln and cur and "attn_kernel" in cur:
            if "0 bytes spill stores, 0 bytes spill loads" not in ln:
                out.append(f"{cur}: {ln.strip()}")
    return out


if __name__ == "__main__":
    print(build(force=True, verbose="--verbose" in sys.argv, trace="--trace" in sys.argv))
    if "--trace" not in sys.argv:
        print(build_count(force=True))
