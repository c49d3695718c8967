"""B200-native TriangleMix prefill attention (arxiv 2507.21526) -- Python binding.

Argument marshalling only: every step of the attention runs in the sm_100a
kernels of ``libtriattn.so`` behind the C ABI declared in ``include/triattn.h``.
PyTorch supplies device memory and the current CUDA stream; nothing here
computes attention.  If the library is missing or the device is not a B200 the
calls raise -- there is no CPU or PyTorch fallback.

Function names follow the C ABI:

    triangle_attn_prefill(q, k, v, sink=8, window=512, last_q=128)   # deep layers
    dense_attn_prefill(q, k, v)                                      # shallow layers
    layer_attn_prefill(layer, tri_start, q, k, v, ...)               # TriangleMix rule
    last_rows_attn_prefill(q, k, v, last_q=128)                      # final layer, last rows
    pair_count(seq_len, sink, window, last_q) / schedule_export(...) # introspection

q: [Hq][N][d] bf16 CUDA tensor view (any strides with unit d-stride), k/v:
[Hkv][N][d]; q head h reads kv head h // (Hq/Hkv).
"""
from __future__ import annotations

import ctypes
import os
import threading

__all__ = [
    "TriattnError", "triangle_attn_prefill", "dense_attn_prefill", "layer_attn_prefill",
    "workspace_size", "pair_count", "schedule_export", "abi_version", "release_caches",
    "triangle_attn_prefill_multi", "dense_attn_prefill_multi",
    "triangle_attn_prefill_multicast", "dense_attn_prefill_multicast",
    "library_path", "STATUS", "profile_begin", "set_pdl", "profile_end", "last_rows_attn_prefill",
    "last_rows_workspace_size", "last_rows_schedule_export",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
# TA_LIBRARY may point at the debug-timeline build (libtriattn_trace.so); same kernels.
_SO = os.environ.get("TA_LIBRARY") or os.path.join(_HERE, "libtriattn.so")

STATUS = {0: "TA_OK", 1: "TA_ERR_NULL_ARG", 2: "TA_ERR_EMPTY_SEQUENCE", 3: "TA_ERR_SHAPE",
          4: "TA_ERR_PARAMS", 5: "TA_ERR_UNSUPPORTED", 6: "TA_ERR_WORKSPACE", 7: "TA_ERR_CUDA"}


class TriattnError(RuntimeError):
    def __init__(self, status: int, detail: str):
        super().__init__(f"{STATUS.get(status, status)}: {detail}")
        self.status = status
        self.detail = detail


class _InTensor(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("stride_head", ctypes.c_int64),
                ("stride_token", ctypes.c_int64)]


class _Problem(ctypes.Structure):
    _fields_ = [("q", _InTensor), ("k", _InTensor), ("v", _InTensor), ("o", _InTensor),
                ("lse", ctypes.c_void_p), ("seq_len", ctypes.c_int64),
                ("num_q_heads", ctypes.c_int32), ("num_kv_heads", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("softmax_scale", ctypes.c_float)]


class _Triangle(ctypes.Structure):
    _fields_ = [("sink", ctypes.c_int32), ("window", ctypes.c_int32), ("last_q", ctypes.c_int32)]


_lib = None


def library_path() -> str:
    return _SO


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_SO):
        raise ImportError(f"{_SO} not built: run `python -m paper_2507_21526_b200.build` "
                          "(there is no fallback path)")
    lib = ctypes.CDLL(_SO)
    P, Tp = ctypes.POINTER(_Problem), ctypes.POINTER(_Triangle)
    vp, sz = ctypes.c_void_p, ctypes.c_size_t
    lib.ta_workspace_size.argtypes = [P, Tp]
    lib.ta_workspace_size.restype = sz
    lib.triangle_attn_prefill.argtypes = [P, Tp, vp, sz, vp]
    lib.triangle_attn_prefill.restype = ctypes.c_int
    lib.dense_attn_prefill.argtypes = [P, vp, sz, vp]
    lib.dense_attn_prefill.restype = ctypes.c_int
    lib.triangle_attn_prefill_multi.argtypes = [P, Tp, vp, ctypes.c_int32, vp, sz, vp]
    lib.triangle_attn_prefill_multi.restype = ctypes.c_int
    lib.dense_attn_prefill_multi.argtypes = [P, vp, ctypes.c_int32, vp, sz, vp]
    lib.dense_attn_prefill_multi.restype = ctypes.c_int
    lib.triangle_attn_prefill_multicast.argtypes = [P, Tp, ctypes.POINTER(_InTensor), vp, sz, vp]
    lib.triangle_attn_prefill_multicast.restype = ctypes.c_int
    lib.dense_attn_prefill_multicast.argtypes = [P, ctypes.POINTER(_InTensor), vp, sz, vp]
    lib.dense_attn_prefill_multicast.restype = ctypes.c_int
    lib.ta_layer_attn_prefill.argtypes = [ctypes.c_int32, ctypes.c_int32, P, Tp, vp, sz, vp]
    lib.ta_layer_attn_prefill.restype = ctypes.c_int
    lib.ta_pair_count.argtypes = [ctypes.c_int64, Tp, ctypes.POINTER(ctypes.c_int64)]
    lib.ta_pair_count.restype = ctypes.c_int
    lib.ta_schedule_export.argtypes = [P, Tp, ctypes.c_int32, vp, ctypes.POINTER(sz)]
    lib.ta_schedule_export.restype = ctypes.c_int
    lib.ta_last_rows_workspace_size.argtypes = [P, ctypes.c_int32]
    lib.ta_last_rows_workspace_size.restype = sz
    lib.last_rows_attn_prefill.argtypes = [P, ctypes.c_int32, vp, sz, vp]
    lib.last_rows_attn_prefill.restype = ctypes.c_int
    lib.ta_last_rows_schedule_export.argtypes = [P, ctypes.c_int32, ctypes.c_int32, vp, ctypes.POINTER(sz)]
    lib.ta_last_rows_schedule_export.restype = ctypes.c_int
    lib.ta_status_str.argtypes = [ctypes.c_int]
    lib.ta_status_str.restype = ctypes.c_char_p
    lib.ta_last_error.argtypes = []
    lib.ta_last_error.restype = ctypes.c_char_p
    lib.ta_abi_version.argtypes = []
    lib.ta_abi_version.restype = ctypes.c_int32
    lib.ta_release_caches.argtypes = []
    lib.ta_release_caches.restype = None
    lib.ta_set_pdl.argtypes = [ctypes.c_int32]
    lib.ta_set_pdl.restype = ctypes.c_int32
    lib.ta_profile_begin.argtypes = []
    lib.ta_profile_begin.restype = ctypes.c_int
    lib.ta_profile_end.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64),
                                   ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)]
    lib.ta_profile_end.restype = ctypes.c_int
    _lib = lib
    return lib


def _check(status: int):
    if status != 0:
        raise TriattnError(status, _load().ta_last_error().decode())


def _view(t):
    return _InTensor(t.data_ptr(), t.stride(0), t.stride(1))


def _problem(q, k, v, o, lse, scale):
    p = _Problem()
    p.q, p.k, p.v, p.o = _view(q), _view(k), _view(v), _view(o)
    p.lse = lse.data_ptr() if lse is not None else None
    p.seq_len = q.shape[1]
    p.num_q_heads = q.shape[0]
    p.num_kv_heads = k.shape[0]
    p.head_dim = q.shape[2]
    p.softmax_scale = float(scale)
    return p


def _check_tensors(q, k, v, o, lse, o_rows=None, extra=()):
    import torch
    for name, t in (("q", q), ("k", k), ("v", v), ("o", o)):
        if t.dtype != torch.bfloat16 or t.dim() != 3 or not t.is_cuda or t.stride(2) != 1:
            raise TriattnError(3, f"{name}: need a CUDA bf16 [heads][tokens][d] view, d-stride 1")
    rows = q.shape[1] if o_rows is None else o_rows
    if k.shape != v.shape or q.shape[1:] != k.shape[1:] or tuple(o.shape) != (q.shape[0], rows, q.shape[2]):
        raise TriattnError(3, "q/k/v/o shapes disagree")
    if lse is not None and (lse.dtype != torch.float32 or not lse.is_contiguous()
                            or tuple(lse.shape) != (q.shape[0], rows)):
        raise TriattnError(3, "lse must be contiguous fp32 [Hq][rows of o]")
    # one device for every buffer: the library launches on the current device, which the
    # calls below set to q's (a foreign pointer would fault or silently cross NVLink)
    for name, t in (("k", k), ("v", v), ("o", o), ("lse", lse)) + tuple(
            (f"extra_out[{i}]", t) for i, t in enumerate(extra)):
        if t is not None and t.device != q.device:
            raise TriattnError(3, f"{name} is on {t.device}, q on {q.device}")


class _Call:
    """Device guard + target stream of one call: the current device is q's for the duration
    of the C call, and the default stream is the current stream *of q's device*."""

    def __init__(self, device, stream):
        import torch
        self.device = device
        self.guard = torch.cuda.device(device)
        if stream is None:
            self.stream = torch.cuda.current_stream(device)
        elif isinstance(stream, torch.cuda.Stream):
            self.stream = stream
        else:  # raw cudaStream_t handle
            self.stream = torch.cuda.ExternalStream(int(stream), device=device)

    def __enter__(self):
        self.guard.__enter__()
        return self

    def __exit__(self, *exc):
        return self.guard.__exit__(*exc)

    @property
    def handle(self):
        return self.stream.cuda_stream


# Split-K workspace: one buffer per (device, stream), allocated with that stream current so
# the caching allocator only ever recycles it in that stream's order (calls on different
# streams never share scratch).  Bounded; an evicted buffer returns to its own stream's pool.
_ws_cache: dict = {}
_ws_lock = threading.Lock()
_WS_MAX_ENTRIES = 8


def _workspace(p, tri, call, last_rows=None):
    import torch
    if last_rows is not None:
        need = _load().ta_last_rows_workspace_size(ctypes.byref(p), int(last_rows))
    else:
        need = _load().ta_workspace_size(ctypes.byref(p), ctypes.byref(tri) if tri is not None else None)
    if need == 0:
        return None, 0
    key = (call.device.index, call.stream.cuda_stream)
    with _ws_lock:
        buf = _ws_cache.get(key)
        if buf is None or buf.numel() < need + 256:
            with torch.cuda.stream(call.stream):
                buf = torch.empty(need + 256, dtype=torch.uint8, device=call.device)
            _ws_cache.pop(key, None)
            while len(_ws_cache) >= _WS_MAX_ENTRIES:
                _ws_cache.pop(next(iter(_ws_cache)))
            _ws_cache[key] = buf
    ptr = (buf.data_ptr() + 255) // 256 * 256
    return ptr, need


def triangle_attn_prefill(q, k, v, o=None, *, sink: int = 8, window: int = 512, last_q: int = 128,
                          lse=None, scale: float = 0.0, stream=None):
    """Triangle attention of one deep layer; returns o."""
    import torch
    if o is None:
        o = torch.empty_like(q)
    _check_tensors(q, k, v, o, lse)
    p = _problem(q, k, v, o, lse, scale)
    tri = _Triangle(sink, window, last_q)
    with _Call(q.device, stream) as c:
        ws, need = _workspace(p, tri, c)
        _check(_load().triangle_attn_prefill(ctypes.byref(p), ctypes.byref(tri), ws, need, c.handle))
    return o


def _extra_views(extra_out, like):
    """ctypes array of ta_out_tensor views of the extra destinations (f2), each checked like o."""
    import torch
    n = len(extra_out)
    arr = (_InTensor * max(n, 1))()
    for e, t in enumerate(extra_out):
        if (t.dtype != torch.bfloat16 or t.dim() != 3 or not t.is_cuda or t.stride(2) != 1
                or tuple(t.shape) != tuple(like.shape)):
            raise TriattnError(3, f"extra_out[{e}]: need a CUDA bf16 view shaped like o, d-stride 1")
        arr[e] = _view(t)
    return arr, n


def triangle_attn_prefill_multi(q, k, v, extra_out, o=None, *, sink: int = 8, window: int = 512,
                                last_q: int = 128, lse=None, scale: float = 0.0, stream=None):
    """triangle_attn_prefill whose epilogue also writes every O tile to each tensor of
    extra_out (f2: e.g. this rank's head slice of peer ranks' full-O buffers); returns o."""
    import torch
    if o is None:
        o = torch.empty_like(q)
    _check_tensors(q, k, v, o, lse, extra=tuple(extra_out))
    arr, n = _extra_views(extra_out, o)
    p = _problem(q, k, v, o, lse, scale)
    tri = _Triangle(sink, window, last_q)
    with _Call(q.device, stream) as c:
        ws, need = _workspace(p, tri, c)
        _check(_load().triangle_attn_prefill_multi(ctypes.byref(p), ctypes.byref(tri), arr, n, ws,
                                                   need, c.handle))
    return o


def dense_attn_prefill_multi(q, k, v, extra_out, o=None, *, lse=None, scale: float = 0.0,
                             stream=None):
    """dense_attn_prefill with the f2 extra output destinations; returns o."""
    import torch
    if o is None:
        o = torch.empty_like(q)
    _check_tensors(q, k, v, o, lse, extra=tuple(extra_out))
    arr, n = _extra_views(extra_out, o)
    p = _problem(q, k, v, o, lse, scale)
    with _Call(q.device, stream) as c:
        ws, need = _workspace(p, None, c)
        _check(_load().dense_attn_prefill_multi(ctypes.byref(p), arr, n, ws, need, c.handle))
    return o


def _mc_view(mc_ptr, mc_strides):
    if not mc_ptr:
        raise TriattnError(1, "multicast pointer is NULL")
    sh, st = mc_strides
    return _InTensor(int(mc_ptr), int(sh), int(st))


def triangle_attn_prefill_multicast(q, k, v, mc_ptr: int, mc_strides, o=None, *, sink: int = 8,
                                    window: int = 512, last_q: int = 128, lse=None,
                                    scale: float = 0.0, stream=None):
    """triangle_attn_prefill that also stores every O tile (and the merged last rows) with
    multimem stores to a [Hq][N][d] view at the multicast address mc_ptr (element strides
    mc_strides = (stride_head, stride_token)): f2 over NVLS, one egress per tile."""
    import torch
    if o is None:
        o = torch.empty_like(q)
    _check_tensors(q, k, v, o, lse)
    mc = _mc_view(mc_ptr, mc_strides)
    p = _problem(q, k, v, o, lse, scale)
    tri = _Triangle(sink, window, last_q)
    with _Call(q.device, stream) as c:
        ws, need = _workspace(p, tri, c)
        _check(_load().triangle_attn_prefill_multicast(ctypes.byref(p), ctypes.byref(tri),
                                                       ctypes.byref(mc), ws, need, c.handle))
    return o


def dense_attn_prefill_multicast(q, k, v, mc_ptr: int, mc_strides, o=None, *, lse=None,
                                 scale: float = 0.0, stream=None):
    """dense_attn_prefill with the f2 multicast output view; returns o."""
    import torch
    if o is None:
        o = torch.empty_like(q)
    _check_tensors(q, k, v, o, lse)
    mc = _mc_view(mc_ptr, mc_strides)
    p = _problem(q, k, v, o, lse, scale)
    with _Call(q.device, stream) as c:
        ws, need = _workspace(p, None, c)
        _check(_load().dense_attn_prefill_multicast(ctypes.byref(p), ctypes.byref(mc), ws, need,
                                                    c.handle))
    return o


def dense_attn_prefill(q, k, v, o=None, *, lse=None, scale: float = 0.0, stream=None):
    """Dense causal attention of one shallow layer; returns o."""
    import torch
    if o is None:
        o = torch.empty_like(q)
    _check_tensors(q, k, v, o, lse)
    p = _problem(q, k, v, o, lse, scale)
    with _Call(q.device, stream) as c:
        ws, need = _workspace(p, None, c)
        _check(_load().dense_attn_prefill(ctypes.byref(p), ws, need, c.handle))
    return o


def layer_attn_prefill(layer: int, tri_start: int, q, k, v, o=None, *, sink: int = 8,
                       window: int = 512, last_q: int = 128, lse=None, scale: float = 0.0,
                       stream=None):
    """TriangleMix per-layer dispatch: dense iff layer < tri_start (reading R2)."""
    import torch
    if o is None:
        o = torch.empty_like(q)
    _check_tensors(q, k, v, o, lse)
    p = _problem(q, k, v, o, lse, scale)
    tri = _Triangle(sink, window, last_q)
    with _Call(q.device, stream) as c:
        ws, need = _workspace(p, None if layer < tri_start else tri, c)
        _check(_load().ta_layer_attn_prefill(layer, tri_start, ctypes.byref(p), ctypes.byref(tri), ws,
                                             need, c.handle))
    return o


def last_rows_attn_prefill(q, k, v, o=None, *, last_q: int = 128, lse=None, scale: float = 0.0,
                           stream=None):
    """Final-layer attention of the last r = min(last_q, N) query rows only:
    o[h, t] = softmax over all causal keys of query N - r + t.  Returns o [Hq][r][d]."""
    import torch
    r = min(int(last_q), q.shape[1]) if last_q >= 1 else int(last_q)
    if o is None:
        o = torch.empty((q.shape[0], max(r, 0), q.shape[2]), dtype=q.dtype, device=q.device)
    _check_tensors(q, k, v, o, lse, o_rows=max(r, 0))
    p = _problem(q, k, v, o, lse, scale)
    with _Call(q.device, stream) as c:
        ws, need = _workspace(p, None, c, last_rows=last_q)
        _check(_load().last_rows_attn_prefill(ctypes.byref(p), int(last_q), ws, need, c.handle))
    return o


def last_rows_workspace_size(seq_len: int, hq: int, hkv: int, d: int, last_q: int = 128) -> int:
    p = _shape_problem(seq_len, hq, hkv, d)
    return int(_load().ta_last_rows_workspace_size(ctypes.byref(p), int(last_q)))


def last_rows_schedule_export(seq_len: int, hq: int, hkv: int, d: int, num_ctas: int,
                              last_q: int = 128) -> bytes:
    p = _shape_problem(seq_len, hq, hkv, d)
    n = ctypes.c_size_t(0)
    lib = _load()
    st = lib.ta_last_rows_schedule_export(ctypes.byref(p), int(last_q), num_ctas, None, ctypes.byref(n))
    if st not in (0, 6):
        _check(st)
    buf = ctypes.create_string_buffer(n.value)
    _check(lib.ta_last_rows_schedule_export(ctypes.byref(p), int(last_q), num_ctas, buf, ctypes.byref(n)))
    return buf.raw[: n.value]


def _shape_problem(seq_len, hq, hkv, d):
    p = _Problem()
    p.seq_len, p.num_q_heads, p.num_kv_heads, p.head_dim = seq_len, hq, hkv, d
    return p


def workspace_size(seq_len: int, hq: int, hkv: int, d: int, sink=8, window=512, last_q=128,
                   dense: bool = False) -> int:
    p = _shape_problem(seq_len, hq, hkv, d)
    tri = None if dense else _Triangle(sink, window, last_q)
    return int(_load().ta_workspace_size(ctypes.byref(p), ctypes.byref(tri) if tri else None))


def pair_count(seq_len: int, sink=8, window=512, last_q=128, dense: bool = False) -> int:
    out = ctypes.c_int64()
    tri = None if dense else _Triangle(sink, window, last_q)
    _check(_load().ta_pair_count(seq_len, ctypes.byref(tri) if tri else None, ctypes.byref(out)))
    return out.value


def schedule_export(seq_len: int, hq: int, hkv: int, d: int, num_ctas: int, sink=8, window=512,
                    last_q=128, dense: bool = False) -> bytes:
    p = _shape_problem(seq_len, hq, hkv, d)
    tri = None if dense else _Triangle(sink, window, last_q)
    tp = ctypes.byref(tri) if tri else None
    n = ctypes.c_size_t(0)
    lib = _load()
    st = lib.ta_schedule_export(ctypes.byref(p), tp, num_ctas, None, ctypes.byref(n))
    if st not in (0, 6):
        _check(st)
    buf = ctypes.create_string_buffer(n.value)
    _check(lib.ta_schedule_export(ctypes.byref(p), tp, num_ctas, buf, ctypes.byref(n)))
    return buf.raw[: n.value]


def abi_version() -> int:
    return int(_load().ta_abi_version())


def release_caches() -> None:
    _load().ta_release_caches()


def set_pdl(on: bool) -> bool:
    """Launch the LSE merge with programmatic dependent launch (default on); returns the
    previous setting."""
    return bool(_load().ta_set_pdl(1 if on else 0))


def profile_begin() -> None:
    """Start recording CUDA events around every attention / merge kernel launch."""
    _check(_load().ta_profile_begin())


def profile_end() -> dict:
    """Stop recording; returns summed device ms and launch counts per kernel."""
    a, m = ctypes.c_double(), ctypes.c_double()
    na, nm = ctypes.c_int64(), ctypes.c_int64()
    _check(_load().ta_profile_end(ctypes.byref(a), ctypes.byref(na), ctypes.byref(m), ctypes.byref(nm)))
    return {"attn_ms": a.value, "attn_launches": na.value, "merge_ms": m.value,
            "merge_launches": nm.value}
