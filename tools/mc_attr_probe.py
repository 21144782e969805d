"""Does this box support NVLink multicast (NVLS)?  Device attributes + a
POSIX-fd multicast object create/export in one process."""
from cuda.bindings import driver as d

def ok(r):
    if r[0] != d.CUresult.CUDA_SUCCESS:
        raise RuntimeError(str(r[0]))
    return r[1:] if len(r) > 2 else (r[1] if len(r) == 2 else None)

ok(d.cuInit(0))
n = ok(d.cuDeviceGetCount())
for i in range(n):
    dev = ok(d.cuDeviceGet(i))
    a = lambda x: ok(d.cuDeviceGetAttribute(x, dev))
    A = d.CUdevice_attribute
    print(i, "multicast", a(A.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED),
          "posix_fd", a(A.CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED),
          "fabric", a(A.CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED),
          "vmm", a(A.CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED))
dev0 = ok(d.cuDeviceGet(0))
ctx = ok(d.cuDevicePrimaryCtxRetain(dev0))
ok(d.cuCtxSetCurrent(ctx))
prop = d.CUmulticastObjectProp()
prop.numDevices = n
prop.handleTypes = d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
prop.size = 1 << 21
g = ok(d.cuMulticastGetGranularity(prop, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED))
print("mc granularity recommended", g)
prop.size = max(g, 1 << 21)
try:
    mc = ok(d.cuMulticastCreate(prop))
    fd = ok(d.cuMemExportToShareableHandle(mc, d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0))
    print("multicast create + export fd ok", fd)
except Exception as e:
    print("multicast create failed", e)
