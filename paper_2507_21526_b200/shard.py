"""Head sharding of one attention layer across ranks.

Rank r of P owns a kv-head range and the query heads that read it (reading R13: q head
h reads kv head h // G, so a contiguous kv-head range owns a contiguous q-head range):

* P <= Hkv (P | Hkv): kv heads [r*Hkv/P, (r+1)*Hkv/P) and all their G q heads;
* P > Hkv (Hkv | P), e.g. Qwen2.5-7B (Hkv = 4) on 8 GPUs: s = P/Hkv
  ranks share kv head r // s and split its G q heads into s contiguous parts
  [floor(i G / s), floor((i+1) G / s)) (Qwen: 3 + 4); each rank runs the kernel with its
  own GQA group (T = 128 // G_local rows per token).

No data-path collective is needed inside attention; the only exchange is the all-gather
of the head-major output (padded to equal shards when the parts are uneven).
Plumbing only: no attention math.
"""
from __future__ import annotations


def head_plan(hq: int, hkv: int, world: int) -> list[tuple[int, int, int, int]]:
    """Per rank (kv0, kv1, q0, q1): kv heads [kv0, kv1) and q heads [q0, q1)."""
    if world < 1 or hq % hkv != 0:
        raise ValueError("bad head counts")
    g = hq // hkv
    if world <= hkv:
        if hkv % world != 0:
            raise ValueError(f"num_kv_heads={hkv} must be divisible by world size {world}")
        per = hkv // world
        return [(r * per, (r + 1) * per, r * per * g, (r + 1) * per * g) for r in range(world)]
    if world % hkv != 0:
        raise ValueError(f"world size {world} must divide or be a multiple of num_kv_heads={hkv}")
    s = world // hkv
    if s > g:
        raise ValueError(f"{s} ranks per kv head > {g} query heads per kv head")
    plan = []
    for r in range(world):
        kvh, i = divmod(r, s)
        plan.append((kvh, kvh + 1, kvh * g + (i * g) // s, kvh * g + ((i + 1) * g) // s))
    return plan


def kv_head_range(hkv: int, rank: int, world: int) -> tuple[int, int]:
    if world < 1 or hkv % world != 0:
        raise ValueError(f"num_kv_heads={hkv} must be divisible by world size {world}")
    per = hkv // world
    return rank * per, (rank + 1) * per


def shard_qkv(q, k, v, rank: int, world: int):
    """Slice [H][N][d] tensors to this rank's heads (views; call .contiguous() to copy)."""
    hq, hkv = q.shape[0], k.shape[0]
    kv0, kv1, q0, q1 = head_plan(hq, hkv, world)[rank]
    return q[q0:q1], k[kv0:kv1], v[kv0:kv1]


def gather_heads(o_shard, world: int, out=None, group=None, plan=None):
    """All-gather head-major shards into [Hq][N][d] on every rank.

    plan: head_plan(...) when the shards may be uneven (P > Hkv); shards are then padded
    to the largest part for all_gather_into_tensor and the padding is dropped."""
    import torch
    import torch.distributed as dist
    if plan is None:
        sizes = [o_shard.shape[0]] * world
    else:
        sizes = [q1 - q0 for (_, _, q0, q1) in plan]
    hq = sum(sizes)
    if out is None:
        out = torch.empty((hq,) + tuple(o_shard.shape[1:]), dtype=o_shard.dtype, device=o_shard.device)
    if world == 1:
        out.copy_(o_shard)
        return out
    m = max(sizes)
    if all(s == m for s in sizes):
        dist.all_gather_into_tensor(out, o_shard.contiguous(), group=group)
        return out
    send = torch.zeros((m,) + tuple(o_shard.shape[1:]), dtype=o_shard.dtype, device=o_shard.device)
    send[: o_shard.shape[0]].copy_(o_shard)
    buf = torch.empty((m * world,) + tuple(o_shard.shape[1:]), dtype=o_shard.dtype, device=o_shard.device)
    dist.all_gather_into_tensor(buf, send, group=group)
    h = 0
    for r, s in enumerate(sizes):
        out[h:h + s].copy_(buf[r * m:r * m + s])
        h += s
    return out
