"""Synthetic-weight Llama-shaped prefill: the structure of the paper's
TTFT measurement (tab:efficiency_ttft) on random weights.

Per layer: RMSNorm -> QKV projection -> RoPE -> attention -> o_proj -> residual ->
RMSNorm -> SwiGLU MLP -> residual.  The GEMMs, norms and RoPE are plain PyTorch/cuBLAS
(library work outside the method); the attention of every layer goes through this
package's C ABI with the TriangleMix layer rule (reading R2): dense for
layer < tri_start, triangle (sink / window / last_q) after.  Q/K/V are consumed straight
from the token-major projection output ([N][H][d] strided views) and O is written
token-major, so no permutes sit between the GEMMs and the attention kernels.  The last
layer may use the final-layer last-rows mode.  No attention math here.
"""
from __future__ import annotations

from dataclasses import dataclass

import paper_2507_21526_b200 as ta


@dataclass
class ModelShape:
    name: str
    hidden: int
    hq: int
    hkv: int
    d: int
    inter: int
    layers: int
    tri_start: int
    rope_theta: float = 500000.0


LLAMA31_8B = ModelShape("llama-3.1-8b", 4096, 32, 8, 128, 14336, 32, 16)
QWEN25_7B = ModelShape("qwen2.5-7b", 3584, 28, 4, 128, 18944, 28, 20, 1000000.0)


class SyntheticPrefill:
    """One set of random layer weights reused by every layer (cost depends on shapes only)."""

    def __init__(self, shape: ModelShape, device, seed: int = 0, dtype=None):
        import torch
        dtype = dtype or torch.bfloat16
        self.s = shape
        g = torch.Generator(device="cpu").manual_seed(seed)
        h, d = shape.hidden, shape.d
        nq, nkv = shape.hq * d, shape.hkv * d

        def w(o, i):
            return (torch.randn(o, i, generator=g) * (1.0 / i ** 0.5)).to(dtype).to(device)

        self.w_qkv = w(nq + 2 * nkv, h)
        self.w_o = w(h, nq)
        self.w_gu = w(2 * shape.inter, h)
        self.w_down = w(h, shape.inter)
        self.device = device
        self.dtype = dtype
        self._rope = {}

    def rope_tables(self, n: int):
        import torch
        if n not in self._rope:
            d = self.s.d
            inv = 1.0 / (self.s.rope_theta ** (torch.arange(0, d, 2, dtype=torch.float64) / d))
            ang = torch.arange(n, dtype=torch.float64)[:, None] * inv[None, :]
            self._rope[n] = (ang.cos().float().to(self.device), ang.sin().float().to(self.device))
        return self._rope[n]

    @staticmethod
    def _rms(x, eps=1e-5):
        import torch
        xf = x.float()
        return (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps)).to(x.dtype)

    def _rope_apply(self, t, cos, sin):
        # t: [N][H][d] (rotate-half convention)
        import torch
        half = t.shape[-1] // 2
        tf = t.float()
        a, b = tf[..., :half], tf[..., half:]
        c, s = cos[:, None, :], sin[:, None, :]
        return torch.cat((a * c - b * s, b * c + a * s), dim=-1).to(t.dtype)

    def forward(self, x, mode: str = "trianglemix", sink: int = 8, window: int = 512,
                last_q: int = 128, final_last_rows: bool = False):
        """x: [N][hidden] bf16 on the device.  mode: 'dense' (every layer dense causal) or
        'trianglemix' (dense below tri_start, triangle after).  Returns the hidden states
        of the last `last_q` tokens after the last layer."""
        import torch
        import torch.nn.functional as F
        s = self.s
        n = x.shape[0]
        nq, nkv = s.hq * s.d, s.hkv * s.d
        cos, sin = self.rope_tables(n)
        tri_start = s.layers if mode == "dense" else s.tri_start
        for layer in range(s.layers):
            h = self._rms(x)
            qkv = F.linear(h, self.w_qkv)                                   # [N][nq + 2 nkv]
            q = self._rope_apply(qkv[:, :nq].view(n, s.hq, s.d), cos, sin)   # [N][Hq][d]
            k = self._rope_apply(qkv[:, nq:nq + nkv].view(n, s.hkv, s.d), cos, sin)
            v = qkv[:, nq + nkv:].view(n, s.hkv, s.d)
            qh, kh, vh = q.transpose(0, 1), k.transpose(0, 1), v.transpose(0, 1)  # strided views
            last_layer = layer == s.layers - 1
            if last_layer and final_last_rows:
                # only the last rows feed the first generated token
                r = min(last_q, n)
                o_last = torch.empty((r, s.hq, s.d), dtype=x.dtype, device=x.device)
                ta.last_rows_attn_prefill(qh, kh, vh, o_last.transpose(0, 1), last_q=r)
                x = x[n - r:]
                attn = o_last.reshape(r, nq)
            else:
                o = torch.empty((n, s.hq, s.d), dtype=x.dtype, device=x.device)
                ta.layer_attn_prefill(layer, tri_start, qh, kh, vh, o.transpose(0, 1), sink=sink,
                                      window=window, last_q=last_q)
                attn = o.view(n, nq)
            x = x + F.linear(attn, self.w_o)
            h = self._rms(x)
            gu = F.linear(h, self.w_gu)
            gate, up = gu[:, :s.inter], gu[:, s.inter:]
            x = x + F.linear(F.silu(gate) * up, self.w_down)
        return x[-min(last_q, x.shape[0]):]
