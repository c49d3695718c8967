"""f2 plumbing on one GPU: the *_multi epilogue storing into a torch symmetric-memory buffer
(the mapping the multi-GPU bench uses for peer ranks' full-O buffers), world size 1, the
peer view being rank 0's own buffer through get_buffer.  Skips if symmetric memory is not
available on the box."""
import os
import socket

import pytest
import torch

import paper_2507_21526_b200 as ta
import synth

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_multi_into_symmetric_memory():
    import torch.distributed as dist
    try:
        import torch.distributed._symmetric_memory as symm
    except ImportError:
        pytest.skip("no torch symmetric memory")
    dev = torch.device("cuda", 0)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        hq, hkv, n, d = 32, 8, 1500, 128
        q, k, v = (t.to(dev) for t in synth.make_qkv(hq, hkv, n, d, 5, "iid", 8))
        try:
            buf = symm.empty((2, hq, n, d), dtype=torch.bfloat16, device=dev)
            hdl = symm.rendezvous(buf, dist.group.WORLD)
            peer = hdl.get_buffer(0, (2, hq, n, d), torch.bfloat16)
        except Exception as e:  # noqa: BLE001
            pytest.skip(f"symmetric memory unavailable: {e}")
        buf.fill_(float("nan"))
        ref = ta.triangle_attn_prefill(q, k, v)
        ta.triangle_attn_prefill_multi(q, k, v, [peer[1]], buf[0])
        hdl.barrier(channel=0)
        torch.cuda.synchronize()
        assert torch.equal(buf[0], ref) and torch.equal(buf[1], ref)
    finally:
        dist.destroy_process_group()
