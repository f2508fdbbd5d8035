"""Probe NVLS multicast through the CUDA driver on this box (f4 multimem
epilogue): device attribute, granularity, and a 1-device multicast object
bound to local memory and mapped.  Prints one JSON line; if the mapping works,
also writes the multicast and unicast addresses' behaviour check result.
python tools/probe_mc_driver.py"""
import json

from cuda.bindings import driver as d


def ok(r):
    err = r[0] if isinstance(r, tuple) else r
    return err == d.CUresult.CUDA_SUCCESS, (r[1] if isinstance(r, tuple) and len(r) > 1 else None)


res = {}
d.cuInit(0)
_, dev = d.cuDeviceGet(0)
_, ctx = d.cuDevicePrimaryCtxRetain(dev)
d.cuCtxSetCurrent(ctx)
e, v = d.cuDeviceGetAttribute(d.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)
res["multicast_supported_attr"] = int(v) if e == d.CUresult.CUDA_SUCCESS else str(e)
prop = d.CUmulticastObjectProp()
prop.numDevices = 1
prop.size = 2 << 20
prop.handleTypes = d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_NONE
e, gran = d.cuMulticastGetGranularity(prop, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
res["granularity"] = int(gran) if e == d.CUresult.CUDA_SUCCESS else str(e)
if e == d.CUresult.CUDA_SUCCESS:
    prop.size = max(int(gran), 2 << 20)
    for ht in (d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_NONE,
               d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
               d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_FABRIC):
        prop.handleTypes = ht
        e, mc = d.cuMulticastCreate(prop)
        res[f"create_{int(ht)}"] = str(e)
        if e == d.CUresult.CUDA_SUCCESS:
            break
    res["create"] = str(e)
    if e == d.CUresult.CUDA_SUCCESS:
        res["add_device"] = str(d.cuMulticastAddDevice(mc, dev)[0])
        ap = d.CUmemAllocationProp()
        ap.type = d.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        ap.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        ap.location.id = 0
        e2, mem = d.cuMemCreate(prop.size, ap, 0)
        res["mem_create"] = str(e2)
        if e2 == d.CUresult.CUDA_SUCCESS:
            res["bind"] = str(d.cuMulticastBindMem(mc, 0, mem, 0, prop.size, 0)[0])
            e3, va = d.cuMemAddressReserve(prop.size, int(gran), 0, 0)
            res["reserve"] = str(e3)
            res["map"] = str(d.cuMemMap(va, prop.size, 0, mc, 0)[0])
            acc = d.CUmemAccessDesc()
            acc.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
            acc.location.id = 0
            acc.flags = d.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
            res["set_access"] = str(d.cuMemSetAccess(va, prop.size, [acc], 1)[0])
print(json.dumps(res))
