"""ctypes loader for attn_oracle.c (plain C fp64 oracle).  TEST INFRASTRUCTURE.

build() compiles it with gcc -O2 -fopenmp; __graft_entry__.build() calls this
("building the checker is not using it").
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "attn_oracle.c")
_SO = os.path.join(_HERE, "_attn_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", _SO, _SRC, "-lm"])
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        p = ctypes.c_void_p
        i64 = ctypes.c_int64
        lib.oracle_attention.argtypes = [p, p, p, i64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         i64, i64, i64, ctypes.c_int, ctypes.c_double, p, i64,
                                         p, p, ctypes.c_int]
        lib.oracle_attention.restype = ctypes.c_int
        lib.oracle_pair_count.argtypes = [i64, i64, i64, i64, ctypes.c_int]
        lib.oracle_pair_count.restype = i64
        _lib = lib
    return _lib


def _bits(x) -> np.ndarray:
    """bf16 torch tensor or uint16 array -> contiguous uint16 numpy array of the bits."""
    if isinstance(x, np.ndarray):
        assert x.dtype == np.uint16
        return np.ascontiguousarray(x)
    import torch  # local: only for the dtype conversion of torch inputs
    assert x.dtype == torch.bfloat16
    return x.contiguous().view(torch.int16).numpy().view(np.uint16)


def attention(q, k, v, si: int, sl: int, last: int, dense: bool, scale: float | None = None,
              rows=None, threads: int = 0):
    """q (Hq,N,d), k/v (Hkv,N,d) bf16 -> (O fp64 (Hq,nrows,d), lse (Hq,nrows), threads used)."""
    lib = _load()
    qb, kb, vb = _bits(q), _bits(k), _bits(v)
    hq, n, d = qb.shape
    hkv = kb.shape[0]
    if scale is None:
        scale = 1.0 / np.sqrt(d)
    if rows is not None:
        rows = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
        nrows = len(rows)
    else:
        nrows = n
    o = np.empty((hq, nrows, d), dtype=np.float64)
    lse = np.empty((hq, nrows), dtype=np.float64)
    used = lib.oracle_attention(
        qb.ctypes.data, kb.ctypes.data, vb.ctypes.data, n, hq, hkv, d, si, sl, last,
        int(dense), float(scale), rows.ctypes.data if rows is not None else None, nrows,
        o.ctypes.data, lse.ctypes.data, int(threads))
    if used < 0:
        raise ValueError("oracle_attention: bad arguments")
    return o, lse, used


def pair_count(n: int, si: int, sl: int, last: int, dense: bool) -> int:
    return int(_load().oracle_pair_count(n, si, sl, last, int(dense)))
