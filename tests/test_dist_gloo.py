"""World-size-2 gloo tests of the KV-head sharding + output all-gather (CPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import cref
from paper_2507_21526_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    hq, hkv, n, d, si, sl, last = cfg
    q, k, v = synth.make_qkv(hq, hkv, n, d, seed=77)
    qs, ks, vs = shard.shard_qkv(q, k, v, rank, world)
    o, _, _ = cref.attention(qs.contiguous(), ks.contiguous(), vs.contiguous(), si, sl, last, False)
    full = shard.gather_heads(torch.from_numpy(o).float(), world, plan=shard.head_plan(hq, hkv, world))
    if rank == 0:
        ret.put(full.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [(8, 4, 300, 32, 4, 40, 30), (28, 4, 200, 16, 8, 64, 16),
                                 (7, 1, 150, 16, 8, 32, 20)])   # Qwen-like group split 3 + 4
def test_sharded_equals_unsharded(cfg):
    world = 2
    ctx = mp.get_context("spawn")
    ret = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, ret)) for r in range(world)]
    for p in procs:
        p.start()
    got = ret.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    hq, hkv, n, d, si, sl, last = cfg
    q, k, v = synth.make_qkv(hq, hkv, n, d, seed=77)
    ref, _, _ = cref.attention(q, k, v, si, sl, last, False)
    assert np.abs(got - ref).max() < 1e-6   # fp32 transport of fp64 results


def test_kv_head_ranges():
    assert [shard.kv_head_range(8, r, 8) for r in range(8)] == [(i, i + 1) for i in range(8)]
    assert shard.kv_head_range(8, 1, 2) == (4, 8)
    with pytest.raises(ValueError):
        shard.kv_head_range(4, 0, 8)   # Qwen (Hkv=4) shards to at most 4 ranks
    q, k, v = synth.make_qkv(32, 8, 4, 8, seed=1)
    qs, ks, vs = shard.shard_qkv(q, k, v, 3, 4)
    assert torch.equal(qs, q[24:32]) and torch.equal(ks, k[6:8])


def test_schedule_per_shard_is_a_kv_head_slice():
    """A shard's schedule equals the full schedule restricted to its kv heads (same items)."""
    import paper_2507_21526_b200 as ta
    from oracle import schedule_ref
    _, _, items_full = schedule_ref.parse(ta.schedule_export(4096, 32, 8, 128, 148))
    _, _, items_shard = schedule_ref.parse(ta.schedule_export(4096, 4, 1, 128, 148))
    stream_full = sorted((p, kb, ke) for kind, kvh, p, kb, ke, _ in items_full if kvh == 0 and kind == 0)
    stream_shard = sorted((p, kb, ke) for kind, kvh, p, kb, ke, _ in items_shard if kind == 0)
    assert stream_full == stream_shard


def test_head_plan_qwen_on_8():
    """Qwen2.5-7B (Hq 28, Hkv 4) on 8 ranks: two ranks per kv head, q heads split 3 + 4."""
    plan = shard.head_plan(28, 4, 8)
    assert plan[0] == (0, 1, 0, 3) and plan[1] == (0, 1, 3, 7) and plan[7] == (3, 4, 24, 28)
    covered = sorted(h for (_, _, a, b) in plan for h in range(a, b))
    assert covered == list(range(28))
    assert all(q0 // 7 == kv0 and (q1 - 1) // 7 == kv0 for (kv0, _, q0, q1) in plan)
    assert shard.head_plan(32, 8, 8) == [(r, r + 1, 4 * r, 4 * r + 4) for r in range(8)]
    with pytest.raises(ValueError):
        shard.head_plan(28, 4, 6)
