"""f2 as specified: the *_multicast entry points store
every O tile and the merged last rows through a multicast (NVLS) virtual address.

One GPU: a multicast object with a single bound device (cuMulticastCreate / AddDevice /
BindMem, CUDA driver API via cuda-python) -- the multimem stores must land in the bound
physical memory exactly like the plain output.  Checked bitwise, through a unicast mapping
of the same physical allocation, against the single-output call, for a head slice at an
offset inside a larger buffer (the layout a rank's slice has in the full-O buffer)."""
import numpy as np
import pytest
import torch

import paper_2507_21526_b200 as ta
import synth
from oracle import cref

pytestmark = pytest.mark.gpu


def _ok(res, what=""):
    from cuda.bindings import driver as cu
    err = res[0] if isinstance(res, tuple) else res
    assert err == cu.CUresult.CUDA_SUCCESS, (what, err)
    if isinstance(res, tuple):
        return res[1] if len(res) == 2 else res[1:]
    return None


class Multicast1:
    """A 1-device multicast object bound to one physical allocation, mapped twice:
    at a multicast VA (mc) and at a unicast VA (uc)."""

    def __init__(self, nbytes, dev=0):
        from cuda.bindings import driver as cu
        self.cu = cu
        torch.cuda.init()
        torch.empty(1, device=f"cuda:{dev}")  # torch's primary context is current
        _ok(cu.cuInit(0))
        d = _ok(cu.cuDeviceGet(dev))
        sup = _ok(cu.cuDeviceGetAttribute(
            cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d))
        if not sup:
            pytest.skip("device reports no multicast (NVLS) support")
        prop = cu.CUmulticastObjectProp()
        prop.numDevices = 1
        prop.size = nbytes
        prop.handleTypes = cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
        gran = _ok(cu.cuMulticastGetGranularity(
            prop, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED), "granularity")
        aprop = cu.CUmemAllocationProp()
        aprop.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        aprop.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        aprop.location.id = dev
        agran = _ok(cu.cuMemGetAllocationGranularity(
            aprop, cu.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_RECOMMENDED))
        g = max(int(gran), int(agran))
        self.size = (nbytes + g - 1) // g * g
        prop.size = self.size
        err, self.mc_handle = cu.cuMulticastCreate(prop)
        if err != cu.CUresult.CUDA_SUCCESS:
            # the 1-GPU gpurun boxes report MULTICAST_SUPPORTED = 1 but refuse every
            # multicast object (profiles/r02_mc_probe.txt, scripts/mc_probe.py)
            pytest.skip(f"cuMulticastCreate: {err.name} (no NVLS multicast object on this box)")
        _ok(cu.cuMulticastAddDevice(self.mc_handle, d), "add device")
        self.mem = _ok(cu.cuMemCreate(self.size, aprop, 0), "mem create")
        _ok(cu.cuMulticastBindMem(self.mc_handle, 0, self.mem, 0, self.size, 0), "bind")
        acc = cu.CUmemAccessDesc()
        acc.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        acc.location.id = dev
        acc.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        self.uc = _ok(cu.cuMemAddressReserve(self.size, g, 0, 0), "reserve uc")
        _ok(cu.cuMemMap(self.uc, self.size, 0, self.mem, 0), "map uc")
        _ok(cu.cuMemSetAccess(self.uc, self.size, [acc], 1), "access uc")
        self.mc = _ok(cu.cuMemAddressReserve(self.size, g, 0, 0), "reserve mc")
        _ok(cu.cuMemMap(self.mc, self.size, 0, self.mc_handle, 0), "map mc")
        _ok(cu.cuMemSetAccess(self.mc, self.size, [acc], 1), "access mc")

    def fill_from(self, t):  # torch tensor -> unicast mapping
        _ok(self.cu.cuMemcpyDtoD(self.uc, t.data_ptr(), t.numel() * t.element_size()))

    def read_into(self, t):  # unicast mapping -> torch tensor
        _ok(self.cu.cuMemcpyDtoD(t.data_ptr(), self.uc, t.numel() * t.element_size()))

    def close(self):
        cu = self.cu
        torch.cuda.synchronize()
        cu.cuMemUnmap(self.mc, self.size)
        cu.cuMemUnmap(self.uc, self.size)
        cu.cuMemAddressFree(self.mc, self.size)
        cu.cuMemAddressFree(self.uc, self.size)
        cu.cuMulticastUnbind(self.mc_handle, 0, 0, self.size)
        cu.cuMemRelease(self.mem)
        cu.cuMemRelease(self.mc_handle)


@pytest.mark.parametrize("dense", [False, True])
def test_multicast_output_bitwise(dense):
    hq, hkv, n, d, si, sl, last = 32, 8, 2049, 128, 8, 512, 128
    q, k, v = synth.make_qkv(hq, hkv, n, d, 21, "iid", si)
    dev = torch.device("cuda")
    qd, kd, vd = q.to(dev), k.to(dev), v.to(dev)
    ref = torch.empty_like(qd)
    if dense:
        ta.dense_attn_prefill(qd, kd, vd, ref)
    else:
        ta.triangle_attn_prefill(qd, kd, vd, ref, sink=si, window=sl, last_q=last)
    # full buffer of 2*hq heads; this "rank" owns heads [hq, 2 hq)
    full = torch.full((2 * hq, n, d), float("nan"), dtype=torch.bfloat16, device=dev)
    mc = Multicast1(full.numel() * 2)
    try:
        mc.fill_from(full)
        torch.cuda.synchronize()
        off = hq * n * d * 2
        o = torch.full_like(qd, float("nan"))
        if dense:
            ta.dense_attn_prefill_multicast(qd, kd, vd, int(mc.mc) + off, (n * d, d), o)
        else:
            ta.triangle_attn_prefill_multicast(qd, kd, vd, int(mc.mc) + off, (n * d, d), o,
                                               sink=si, window=sl, last_q=last)
        torch.cuda.synchronize()
        got = torch.empty_like(full)
        mc.read_into(got)
        torch.cuda.synchronize()
    finally:
        mc.close()
    assert torch.equal(o, ref)
    assert torch.equal(got[hq:], ref)                 # every tile and last row arrived
    assert torch.isnan(got[:hq].float()).all()       # nothing outside the slice
    o_ref, _, _ = cref.attention(q, k, v, si, sl, last, dense)
    err = np.abs(o.float().cpu().double().numpy() - o_ref)
    assert err.max() <= 2e-2 and err.mean() <= 2e-3


@pytest.mark.parametrize("dense", [False, True])
def test_multicast_epilogue_addressing_unicast_standin(dense):
    """The multicast epilogue / merge store path (16-byte multimem.st from the staged tile)
    with an ordinary device buffer standing in for the multicast view: on sm_100a
    multimem.st.global.v4.bf16x2 assembles to the same STG.E.128 as a plain store (the NVLS
    replication is done by the address translation), so this checks every index of the path
    -- head slice at an offset, token-major strides -- bitwise against the single output.
    (Replication itself needs a multicast object: test_multicast_output_bitwise.)"""
    hq, hkv, n, d, si, sl, last = 28, 4, 1500, 128, 8, 512, 128
    q, k, v = synth.make_qkv(hq, hkv, n, d, 22, "iid", si)
    dev = torch.device("cuda")
    qd, kd, vd = q.to(dev), k.to(dev), v.to(dev)
    ref = torch.empty_like(qd)
    if dense:
        ta.dense_attn_prefill(qd, kd, vd, ref)
    else:
        ta.triangle_attn_prefill(qd, kd, vd, ref, sink=si, window=sl, last_q=last)
    big = torch.full((n, 2 * hq, d), float("nan"), dtype=torch.bfloat16, device=dev)  # token-major
    view = big[:, hq:, :]
    o = torch.empty_like(qd)
    ptr, strides = view.data_ptr(), (view.stride(1), view.stride(0))
    if dense:
        ta.dense_attn_prefill_multicast(qd, kd, vd, ptr, strides, o)
    else:
        ta.triangle_attn_prefill_multicast(qd, kd, vd, ptr, strides, o, sink=si, window=sl,
                                           last_q=last)
    torch.cuda.synchronize()
    assert torch.equal(o, ref)
    assert torch.equal(view.permute(1, 0, 2), ref)
    assert torch.isnan(big[:, :hq].float()).all()


def test_multicast_null_is_an_error():
    q, k, v = (torch.zeros((4, 64, 128), dtype=torch.bfloat16, device="cuda") for _ in range(3))
    with pytest.raises(ta.TriattnError) as e:
        ta.triangle_attn_prefill_multicast(q, k[:1], v[:1], 0, (64 * 128, 128))
    assert e.value.status == 1
