"""Seeded synthetic workloads shared by the tests, the bench and the oracle legs.

Holds NONE of the method's arithmetic: only shapes (BASELINE.json configs) and
seeded random Q/K/V in the paper's layout.  Recipe:

* shapes: Llama-3.1-8B attention (Hq=32, Hkv=8, d=128) and Qwen2.5-7B
  (Hq=28, Hkv=4, d=128) at N = 32K/64K/128K = 2^15/2^16/2^17 (reading R15),
  batch 1 (R16); si/sl/last = 8/512/128; C1 is 1 head, d=64, N=512,
  si/sl/last = 4/64/64.
* values: fp32 iid N(0,1) drawn from torch.Generator('cpu').manual_seed(
  1000*cfg + layer) in the fixed order Q (Hq,N,d), K (Hkv,N,d), V (Hkv,N,d),
  then rounded to bf16 (RNE); both the CUDA path and the oracle consume these
  same bf16 values.
* stress variants (parity only): "large" (Q, K x 3), "sink" (sink keys
  shifted along the mean-query direction), "zeroq_onehot" (Q = 0, V one-hot
  V[j, j mod d] = 1), "ones_v" (V = 1).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class Config:
    cid: int
    name: str
    hq: int
    hkv: int
    d: int
    n: int
    si: int
    sl: int
    last: int
    tri_start: int
    n_layers: int


PAPER_TRI = dict(si=8, sl=512, last=128)
CONFIGS = {
    "C1": Config(1, "tiny-1head-d64-N512", 1, 1, 64, 512, 4, 64, 64, 0, 1),
    "C2": Config(2, "llama3.1-8b-attn-N32K", 32, 8, 128, 32768, tri_start=16, n_layers=32,
                 **PAPER_TRI),
    "C3": Config(3, "llama3.1-8b-attn-N128K", 32, 8, 128, 131072, tri_start=16, n_layers=32,
                 **PAPER_TRI),
    "C4a": Config(4, "qwen2.5-7b-attn-N64K", 28, 4, 128, 65536, tri_start=20, n_layers=28,
                  **PAPER_TRI),
    "C4b": Config(4, "qwen2.5-7b-attn-N128K", 28, 4, 128, 131072, tri_start=20, n_layers=28,
                  **PAPER_TRI),
}


def make_qkv(hq: int, hkv: int, n: int, d: int, seed: int, dist: str = "iid", si: int = 8):
    """Return CPU bf16 tensors q (hq,n,d), k (hkv,n,d), v (hkv,n,d)."""
    g = torch.Generator("cpu").manual_seed(int(seed))
    q = torch.randn((hq, n, d), generator=g, dtype=torch.float32)
    k = torch.randn((hkv, n, d), generator=g, dtype=torch.float32)
    v = torch.randn((hkv, n, d), generator=g, dtype=torch.float32)
    if dist == "iid":
        pass
    elif dist == "large":
        q *= 3.0
        k *= 3.0
    elif dist == "sink":
        u = q.mean(dim=(0, 1))
        u = u / u.norm()
        k[:, :si, :] += 80.0 * u
    elif dist == "zeroq_onehot":
        q.zero_()
        v.zero_()
        j = torch.arange(n)
        v[:, j, j % d] = 1.0
    elif dist == "ones_v":
        v.fill_(1.0)
    elif dist == "ramp":
        # scores that grow along every 384-key period by ~80 log2 units: later key blocks
        # of a row exceed the first block's max by far more than any lazy-rescale headroom
        # (exercises the rescale / deferred-max re-run paths; DESIGN reading R15)
        u = torch.randn(d, generator=g)
        u = u / u.norm()
        q = 0.5 * q + 4.0 * u
        a = 160.0 * (torch.arange(n, dtype=torch.float32) % 384) / 384.0
        k = 0.5 * k + a[None, :, None] * u
    else:
        raise ValueError(dist)
    return q.to(torch.bfloat16), k.to(torch.bfloat16), v.to(torch.bfloat16)


def config_qkv(cfg: Config, layer: int = 0, dist: str = "iid"):
    return make_qkv(cfg.hq, cfg.hkv, cfg.n, cfg.d, 1000 * cfg.cid + layer, dist, cfg.si)
