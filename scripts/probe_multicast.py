"""Does this box expose NVLink multicast (NVLS) objects? Prints the device attribute and tries a one-device
multicast object (cuMulticastCreate + AddDevice) — the prerequisite of a multimem.st exchange."""
from cuda.bindings import driver as d

def ok(r):
    return r[0] == d.CUresult.CUDA_SUCCESS

print("cuInit", d.cuInit(0)[0])
dev = d.cuDeviceGet(0)[1]
ctx = d.cuDevicePrimaryCtxRetain(dev)[1]
d.cuCtxSetCurrent(ctx)
r = d.cuDeviceGetAttribute(d.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)
print("MULTICAST_SUPPORTED", r)
p = d.CUmulticastObjectProp()
p.numDevices = 1
p.size = 2 << 20
p.handleTypes = d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
g = d.cuMulticastGetGranularity(p, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
print("granularity", g)
r = d.cuMulticastCreate(p)
print("cuMulticastCreate", r[0])
if ok(r):
    print("cuMulticastAddDevice", d.cuMulticastAddDevice(r[1], dev)[0])
