from cuda.bindings import driver as d
def ok(r):
    if not isinstance(r, tuple): r=(r,)
    return r
print(ok(d.cuInit(0)))
err, dev = d.cuDeviceGet(0)
for a in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED","CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED","CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED"):
    print(a, d.cuDeviceGetAttribute(getattr(d.CUdevice_attribute, a), dev))
err, ctx = d.cuDevicePrimaryCtxRetain(dev); d.cuCtxSetCurrent(ctx)
for ht in ("CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR","CU_MEM_HANDLE_TYPE_FABRIC","CU_MEM_HANDLE_TYPE_NONE"):
  for nd in (1, 2):
    p = d.CUmulticastObjectProp(); p.numDevices = nd; p.size = 512 << 20; p.handleTypes = getattr(d.CUmemAllocationHandleType, ht)
    g = d.cuMulticastGetGranularity(p, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_MINIMUM)
    g2 = d.cuMulticastGetGranularity(p, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
    r = d.cuMulticastCreate(p)
    print(ht, nd, g, g2, r[0])
