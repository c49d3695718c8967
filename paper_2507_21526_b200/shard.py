"""KV-head sharding of one attention layer across ranks.

Rank r of P owns kv heads [r*Hkv/P, (r+1)*Hkv/P) and their G = Hq/Hkv query heads
(reading R13: q head h reads kv head h // G, so a contiguous kv-head range owns a
contiguous q-head range).  No data-path collective is needed inside attention; the only
exchange is the all-gather of the head-major output.  Plumbing only: no attention math.
"""
from __future__ import annotations


def kv_head_range(hkv: int, rank: int, world: int) -> tuple[int, int]:
    if world < 1 or hkv % world != 0:
        raise ValueError(f"num_kv_heads={hkv} must be divisible by world size {world}")
    per = hkv // world
    return rank * per, (rank + 1) * per


def shard_qkv(q, k, v, rank: int, world: int):
    """Slice [H][N][d] tensors to this rank's heads (views; call .contiguous() to copy)."""
    hq, hkv = q.shape[0], k.shape[0]
    if hq % hkv != 0:
        raise ValueError("Hq % Hkv != 0")
    g = hq // hkv
    k0, k1 = kv_head_range(hkv, rank, world)
    return q[k0 * g:k1 * g], k[k0:k1], v[k0:k1]


def gather_heads(o_shard, world: int, out=None, group=None):
    """All-gather head-major shards [Hq/P][N][d] into [Hq][N][d] on every rank."""
    import torch
    import torch.distributed as dist
    if out is None:
        out = torch.empty((o_shard.shape[0] * world,) + tuple(o_shard.shape[1:]),
                          dtype=o_shard.dtype, device=o_shard.device)
    if world == 1:
        out.copy_(o_shard)
        return out
    dist.all_gather_into_tensor(out, o_shard.contiguous(), group=group)
    return out
