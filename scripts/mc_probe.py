"""Probe which multicast-object properties this box's driver accepts (1 GPU)."""
import torch
from cuda.bindings import driver as cu

torch.empty(1, device="cuda")
cu.cuInit(0)
_, d = cu.cuDeviceGet(0)
for attr in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED",
             "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED"):
    a = getattr(cu.CUdevice_attribute, attr, None)
    print(attr, cu.cuDeviceGetAttribute(a, d) if a is not None else "n/a")
HT = cu.CUmemAllocationHandleType
for nd in (1, 2):
    for ht_name in ("CU_MEM_HANDLE_TYPE_NONE", "CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR",
                    "CU_MEM_HANDLE_TYPE_FABRIC"):
        ht = getattr(HT, ht_name, None)
        prop = cu.CUmulticastObjectProp()
        prop.numDevices = nd
        prop.handleTypes = ht if ht is not None else 0
        prop.size = 2 << 20
        for gflag in (cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_MINIMUM,
                      cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED):
            e, g = cu.cuMulticastGetGranularity(prop, gflag)
            prop.size = max(int(g), 2 << 20) if e == cu.CUresult.CUDA_SUCCESS else 2 << 20
            e2, h = cu.cuMulticastCreate(prop)
            print(f"numDevices={nd} {ht_name} gran({gflag.name})={e.name}:{g} size={prop.size} "
                  f"create={e2.name}", flush=True)
            if e2 == cu.CUresult.CUDA_SUCCESS:
                print("   add device:", cu.cuMulticastAddDevice(h, d)[0].name)
                cu.cuMemRelease(h)
