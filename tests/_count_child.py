"""Child process of tests/test_gpu_count.py: runs one call through the TA_COUNT build
(TA_LIBRARY=libtriattn_count.so) and writes the per-row counters to an .npy file."""
import ctypes
import sys

import numpy as np
import torch

import paper_2507_21526_b200 as ta
import synth

mode, hq, hkv, n, si, sl, last, out = sys.argv[1], *map(int, sys.argv[2:8]), sys.argv[8]
q, k, v = (t.cuda() for t in synth.make_qkv(hq, hkv, n, 128, seed=n))
if mode == "dense":
    ta.dense_attn_prefill(q, k, v)
elif mode == "last_rows":
    ta.last_rows_attn_prefill(q, k, v, last_q=last)
else:
    ta.triangle_attn_prefill(q, k, v, sink=si, window=sl, last_q=last)
torch.cuda.synchronize()
lib = ta._load()
lib.ta_debug_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
buf = np.zeros((hq, n, 2), dtype=np.uint32)
assert lib.ta_debug_trace_read(buf.ctypes.data, buf.nbytes) == 0
np.save(out, buf)
