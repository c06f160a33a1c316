"""Probe which multicast-object configurations the driver accepts on this box (NVLS plumbing)."""
from cuda.bindings import driver as d

d.cuInit(0)
err, dev = d.cuDeviceGet(0)
err, ctx = d.cuDevicePrimaryCtxRetain(dev)
d.cuCtxSetCurrent(ctx)
print("MULTICAST_SUPPORTED", d.cuDeviceGetAttribute(d.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev))
HT = d.CUmemAllocationHandleType
for ht_name, ht in [("none", 0), ("posix_fd", HT.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
                    ("fabric", HT.CU_MEM_HANDLE_TYPE_FABRIC)]:
    for nd in (1, 2):
        p = d.CUmulticastObjectProp()
        p.numDevices = nd
        p.handleTypes = ht
        p.size = 2 << 20
        e, g = d.cuMulticastGetGranularity(p, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
        p.size = max(g or 0, 2 << 20)
        e2, mc = d.cuMulticastCreate(p)
        res = [str(e), g, str(e2)]
        if e2 == d.CUresult.CUDA_SUCCESS:
            res.append(str(d.cuMulticastAddDevice(mc, dev)[0] if isinstance(d.cuMulticastAddDevice(mc, dev), tuple) else d.cuMulticastAddDevice(mc, dev)))
        print(ht_name, nd, res)
