"""C-ABI boundary on CPU: the library loads, exports every symbol include/triattn.h
declares, and its host-only entry points validate arguments (no GPU compute)."""
import ctypes
import os
import re

import pytest

import paper_2507_21526_b200 as ta
from oracle import counts

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "triattn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*([a-z_0-9]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    names = _declared_functions()
    assert {"triangle_attn_prefill", "dense_attn_prefill", "ta_layer_attn_prefill",
            "ta_workspace_size", "ta_pair_count", "ta_schedule_export"} <= set(names)
    lib = ctypes.CDLL(ta.library_path())
    for nm in names:
        assert hasattr(lib, nm), nm


def test_abi_version():
    assert ta.abi_version() == 4


def test_status_strings():
    lib = ta._load()
    for code, name in ta.STATUS.items():
        assert lib.ta_status_str(code).decode() == name


@pytest.mark.parametrize("n,si,sl,last", [(512, 4, 64, 64), (32768, 8, 512, 128),
                                          (131072, 8, 512, 128), (1, 8, 512, 128),
                                          (100, 0, 1, 1), (777, 30, 5, 1000),
                                          (4096, 8, 512, 0)])
def test_pair_count_matches_oracle(n, si, sl, last):
    assert ta.pair_count(n, si, sl, last) == counts.triangle_pairs(n, si, sl, last)
    assert ta.pair_count(n, dense=True) == counts.dense_pairs(n)


def test_pair_count_paper_values():
    # closed-form values at the paper configuration (derived from P:L295)
    assert ta.pair_count(32768) == 21024036
    assert ta.pair_count(131072) == 84725028
    assert ta.pair_count(512, 4, 64, 64) == 58938


def test_pair_count_errors():
    with pytest.raises(ta.TriattnError) as e:
        ta.pair_count(0)
    assert e.value.status == 2
    with pytest.raises(ta.TriattnError) as e:
        ta.pair_count(10, 8, 0, 128)
    assert e.value.status == 4
    with pytest.raises(ta.TriattnError) as e:
        ta.pair_count(10, -1, 5, 128)
    assert e.value.status == 4
    with pytest.raises(ta.TriattnError) as e:
        ta.pair_count(10, 1, 5, -1)
    assert e.value.status == 4
    # last_q = 0 (StreamingMix) is valid: the streaming count alone
    assert ta.pair_count(100, 4, 10, 0) == counts.streaming_pairs(100, 4, 10)


def test_schedule_export_errors():
    with pytest.raises(ta.TriattnError) as e:
        ta.schedule_export(0, 32, 8, 128, 148)
    assert e.value.status == 2
    with pytest.raises(ta.TriattnError) as e:
        ta.schedule_export(100, 30, 8, 128, 148)
    assert e.value.status == 3
    with pytest.raises(ta.TriattnError) as e:
        ta.schedule_export(100, 32, 8, 96, 148)
    assert e.value.status == 5
    with pytest.raises(ta.TriattnError) as e:
        ta.schedule_export(100, 32, 8, 128, 0)
    assert e.value.status == 4


def test_last_rows_validation():
    with pytest.raises(ta.TriattnError) as e:
        ta.last_rows_schedule_export(100, 32, 8, 128, 148, 0)
    assert e.value.status == 4
    assert ta.last_rows_workspace_size(100, 32, 8, 128, 0) == 0
    assert ta.last_rows_workspace_size(131072, 32, 8, 128, 128) > 0
    lib = ta._load()
    p = ta._shape_problem(64, 32, 8, 128)
    assert lib.last_rows_attn_prefill(ctypes.byref(p), 0, None, 0, None) == 4
    assert lib.last_rows_attn_prefill(ctypes.byref(p), 16, None, 0, None) == 1  # NULL data


def test_workspace_size():
    # every call needs the 256-byte work-queue block; triangle adds the split-K partials
    assert ta.workspace_size(32768, 32, 8, 128, dense=True) == 256
    w = ta.workspace_size(32768, 32, 8, 128)
    assert w > 256 and w % 256 == 0
    assert ta.workspace_size(0, 32, 8, 128) == 0


def test_launch_validation_without_gpu():
    """Null / bad problems are rejected before any CUDA call."""
    lib = ta._load()
    assert lib.triangle_attn_prefill(None, None, None, 0, None) == 1
    p = ta._shape_problem(0, 32, 8, 128)
    tri = ta._Triangle(8, 512, 128)
    assert lib.triangle_attn_prefill(ctypes.byref(p), ctypes.byref(tri), None, 0, None) == 2
    p = ta._shape_problem(64, 32, 8, 128)  # data pointers are NULL
    assert lib.triangle_attn_prefill(ctypes.byref(p), ctypes.byref(tri), None, 0, None) == 1
    assert "q.data" in lib.ta_last_error().decode()
    assert lib.ta_layer_attn_prefill(-1, 16, ctypes.byref(p), ctypes.byref(tri), None, 0, None) == 4


def test_no_cpu_fallback_in_product():
    """The product package never imports the oracle or computes attention in Python."""
    pkg = os.path.join(ROOT, "paper_2507_21526_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            s = open(os.path.join(pkg, f)).read()
            assert not re.search(r"^\s*(from|import)\s+oracle", s, flags=re.M), f
            for bad in ("scaled_dot_product_attention", ".softmax(", "torch.exp(", "np.exp("):
                assert bad not in s, (f, bad)


def test_graft_entry_build():
    """The driver's build() check: compiles (or finds current) libraries and checks the ABI."""
    import importlib
    import sys
    sys.path.insert(0, ROOT)
    g = importlib.import_module("__graft_entry__")
    g.build()


def test_multi_destination_validation_without_gpu():
    """f2 entry points: n_extra range and NULL destinations are rejected before any CUDA call."""
    lib = ta._load()
    p = ta._shape_problem(64, 32, 8, 128)
    fake = 1 << 20  # aligned, never dereferenced on the host
    for t in ("q", "o"):
        setattr(p, t, ta._InTensor(fake, 64 * 128, 128))
    for t in ("k", "v"):
        setattr(p, t, ta._InTensor(fake, 64 * 128, 128))
    tri = ta._Triangle(8, 512, 128)
    arr = (ta._InTensor * 8)(*[ta._InTensor(fake, 64 * 128, 128) for _ in range(8)])
    assert lib.triangle_attn_prefill_multi(ctypes.byref(p), ctypes.byref(tri), arr, 8, None, 0, None) == 4
    assert lib.triangle_attn_prefill_multi(ctypes.byref(p), ctypes.byref(tri), arr, -1, None, 0, None) == 4
    assert lib.triangle_attn_prefill_multi(ctypes.byref(p), ctypes.byref(tri), None, 1, None, 0, None) == 1
    arr[0] = ta._InTensor(0, 64 * 128, 128)
    assert lib.dense_attn_prefill_multi(ctypes.byref(p), arr, 1, None, 0, None) == 1
    assert "extra_o" in lib.ta_last_error().decode()
