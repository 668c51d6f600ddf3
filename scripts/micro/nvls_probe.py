"""Probe: can this box create an NVLink multicast (NVLS) object? Prints the device
attributes and the result of cuMulticastCreate / AddDevice / BindMem / MapAddr with
one device (a gpurun lease exposes a single GPU)."""
import json

import torch
from cuda.bindings import driver as d


def ok(r):
    return r[0] == d.CUresult.CUDA_SUCCESS if isinstance(r, tuple) else r == d.CUresult.CUDA_SUCCESS


torch.cuda.init()
torch.zeros(1, device="cuda")
(_,) = d.cuInit(0)
_, dev = d.cuDeviceGet(0)
out = {}
for name in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED",
             "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED"):
    r = d.cuDeviceGetAttribute(getattr(d.CUdevice_attribute, name), dev)
    out[name] = int(r[1]) if ok(r) else str(r[0])
HT = d.CUmemAllocationHandleType
for name, ht in (("none", 0), ("fd", HT.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR), ("fabric", HT.CU_MEM_HANDLE_TYPE_FABRIC)):
    prop = d.CUmulticastObjectProp()
    prop.numDevices = 1
    prop.size = 2 << 20
    prop.handleTypes = ht
    r = d.cuMulticastGetGranularity(prop, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
    out[name + "_granularity"] = int(r[1]) if ok(r) else str(r[0])
    r = d.cuMulticastCreate(prop)
    out[name + "_create"] = str(r[0])
    if not ok(r):
        continue
    mc = r[1]
    out[name + "_add_device"] = str(d.cuMulticastAddDevice(mc, dev)[0])
    ap = d.CUmemAllocationProp()
    ap.type = d.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
    ap.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    ap.location.id = 0
    ap.requestedHandleTypes = ht
    r2 = d.cuMemCreate(2 << 20, ap, 0)
    out[name + "_mem_create"] = str(r2[0])
    if ok(r2):
        out[name + "_bind"] = str(d.cuMulticastBindMem(mc, 0, r2[1], 0, 2 << 20, 0)[0])
        r3 = d.cuMemAddressReserve(2 << 20, 2 << 20, 0, 0)
        if ok(r3):
            out[name + "_map_mc"] = str(d.cuMemMap(r3[1], 2 << 20, 0, mc, 0)[0])
    break
print(json.dumps(out))
