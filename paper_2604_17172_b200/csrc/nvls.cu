// nvls.cu -- NVLink SHARP (NVLS) multicast support ("transmitted
// directly between GPUs via NVLink").
//
// On NVSwitch systems a multicast object binds one allocation per GPU at the same offset; a
// `multimem.st` to the object's address is replicated by the switch into every bound allocation.
// The allgather-phase fan-out (one encoded stream to N-1 peers, a10) then leaves the sender once
// instead of N-1 times.  The communicator takes such a mapping from outside (uzip_comm_init_ext:
// e.g. torch.distributed._symmetric_memory's multicast_ptr); this file holds the capability probe
// and a single-GPU self-test of the primitive (a one-device multicast object: create, add device,
// bind, map, store through multimem.st, read back through the unicast mapping).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "uzip_internal.h"

namespace uzip {
namespace {

struct Drv {
  bool ok = false;
  CUresult (*getAttr)(int *, CUdevice_attribute, CUdevice) = nullptr;
  CUresult (*mcCreate)(CUmemGenericAllocationHandle *, const CUmulticastObjectProp *) = nullptr;
  CUresult (*mcAdd)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
  CUresult (*mcBind)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                     unsigned long long) = nullptr;
  CUresult (*mcUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
  CUresult (*mcGran)(size_t *, const CUmulticastObjectProp *, CUmulticastGranularity_flags) = nullptr;
  CUresult (*memCreate)(CUmemGenericAllocationHandle *, size_t, const CUmemAllocationProp *,
                        unsigned long long) = nullptr;
  CUresult (*memRelease)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*addrReserve)(CUdeviceptr *, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*addrFree)(CUdeviceptr, size_t) = nullptr;
  CUresult (*memMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*memUnmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*setAccess)(CUdeviceptr, size_t, const CUmemAccessDesc *, size_t) = nullptr;
  CUresult (*allocGran)(size_t *, const CUmemAllocationProp *, CUmemAllocationGranularity_flags) = nullptr;
};

template <class F>
bool sym(const char *name, F &f) {
  void *p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || !p) return false;
  f = reinterpret_cast<F>(p);
  return true;
}

const Drv &drv() {
  static Drv d = [] {
    Drv x;
    x.ok = sym("cuDeviceGetAttribute", x.getAttr) && sym("cuMulticastCreate", x.mcCreate) &&
           sym("cuMulticastAddDevice", x.mcAdd) && sym("cuMulticastBindMem", x.mcBind) &&
           sym("cuMulticastUnbind", x.mcUnbind) && sym("cuMulticastGetGranularity", x.mcGran) &&
           sym("cuMemCreate", x.memCreate) && sym("cuMemRelease", x.memRelease) &&
           sym("cuMemAddressReserve", x.addrReserve) && sym("cuMemAddressFree", x.addrFree) &&
           sym("cuMemMap", x.memMap) && sym("cuMemUnmap", x.memUnmap) && sym("cuMemSetAccess", x.setAccess) &&
           sym("cuMemGetAllocationGranularity", x.allocGran);
    return x;
  }();
  return d;
}

__global__ void k_mc_store(uint8_t *mc, uint64_t n16, uint32_t salt) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t a = (uint32_t)i * 2654435761u ^ salt;
    mc_store_v4(mc + 16 * i, make_uint4(a, a + 1, a ^ 0x55555555u, ~a));
  }
}

__global__ void k_mc_check(const uint8_t *uc, uint64_t n16, uint32_t salt, uint32_t *bad) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t a = (uint32_t)i * 2654435761u ^ salt;
    const uint4 v = reinterpret_cast<const uint4 *>(uc)[i];
    if (v.x != a || v.y != a + 1 || v.z != (a ^ 0x55555555u) || v.w != ~a) atomicAdd(bad, 1u);
  }
}

}  // namespace
}  // namespace uzip

using namespace uzip;

extern "C" {

uzip_status_t uzip_nvls_supported(int device, int *supported) {
  if (!supported) return UZIP_ERR_INVALID_ARG;
  *supported = 0;
  const Drv &d = drv();
  if (!d.ok) return UZIP_OK;
  int v = 0;
  if (d.getAttr(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, (CUdevice)device) != CUDA_SUCCESS) return UZIP_ERR_CUDA;
  *supported = v;
  return UZIP_OK;
}

uzip_status_t uzip_nvls_selftest(int device, size_t bytes) {
  int sup = 0;
  if (uzip_status_t s = uzip_nvls_supported(device, &sup)) return s;
  if (!sup) return UZIP_ERR_NOT_IMPLEMENTED;
  const Drv &d = drv();
  if (cudaSetDevice(device) != cudaSuccess) return UZIP_ERR_CUDA;
  cudaFree(nullptr);  // the primary context exists
  CUmulticastObjectProp mp;
  memset(&mp, 0, sizeof mp);
  mp.numDevices = 1;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;  // NONE is rejected by cuMulticastCreate
  size_t gran = 0;
  mp.size = bytes;
  if (d.mcGran(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS || !gran) return UZIP_ERR_CUDA;
  CUmemAllocationProp ap;
  memset(&ap, 0, sizeof ap);
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = device;
  size_t agran = 0;
  if (d.allocGran(&agran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS) return UZIP_ERR_CUDA;
  if (agran > gran) gran = agran;
  const size_t size = (bytes + gran - 1) / gran * gran;
  mp.size = size;
  CUmemGenericAllocationHandle mc = 0, mem = 0;
  CUdeviceptr uva = 0, mva = 0;
  uzip_status_t st = UZIP_ERR_CUDA;
  CUmemAccessDesc acc;
  memset(&acc, 0, sizeof acc);
  acc.location = ap.location;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  uint32_t *bad = nullptr, hbad = 1;
  CUresult rc = CUDA_SUCCESS;
  int step = 0;
  if ((rc = d.mcCreate(&mc, &mp)) != CUDA_SUCCESS) {  // the attribute says yes, but this node cannot build
    step = 1;                                          // multicast teams (measured: CUDA_ERROR_INVALID_VALUE
    st = UZIP_ERR_NOT_IMPLEMENTED;                     // in the single-GPU gpurun container)
    goto out;
  }
  if ((rc = d.mcAdd(mc, (CUdevice)device)) != CUDA_SUCCESS) {
    step = 2;
    goto out;
  }
  if ((rc = d.memCreate(&mem, size, &ap, 0)) != CUDA_SUCCESS) {
    step = 3;
    goto out;
  }
  if ((rc = d.mcBind(mc, 0, mem, 0, size, 0)) != CUDA_SUCCESS) {
    step = 4;
    goto out;
  }
  if ((rc = d.addrReserve(&uva, size, gran, 0, 0)) != CUDA_SUCCESS) {
    step = 5;
    goto out;
  }
  if ((rc = d.memMap(uva, size, 0, mem, 0)) != CUDA_SUCCESS) {
    step = 6;
    goto out;
  }
  if ((rc = d.setAccess(uva, size, &acc, 1)) != CUDA_SUCCESS) {
    step = 7;
    goto out;
  }
  if ((rc = d.addrReserve(&mva, size, gran, 0, 0)) != CUDA_SUCCESS) {
    step = 8;
    goto out;
  }
  if ((rc = d.memMap(mva, size, 0, mc, 0)) != CUDA_SUCCESS) {
    step = 9;
    goto out;
  }
  if ((rc = d.setAccess(mva, size, &acc, 1)) != CUDA_SUCCESS) {
    step = 10;
    goto out;
  }
  if (cudaMalloc(&bad, 4) != cudaSuccess || cudaMemset(bad, 0, 4) != cudaSuccess) goto out;
  k_mc_store<<<148, 256>>>(reinterpret_cast<uint8_t *>(mva), size / 16, 0x9E3779B9u);
  k_mc_check<<<148, 256>>>(reinterpret_cast<const uint8_t *>(uva), size / 16, 0x9E3779B9u, bad);
  if (cudaMemcpy(&hbad, bad, 4, cudaMemcpyDeviceToHost) != cudaSuccess) goto out;
  st = hbad == 0 ? UZIP_OK : UZIP_ERR_CORRUPT_STREAM;
out:
  if (step && getenv("UZIP_DEBUG"))
    fprintf(stderr, "uzip_nvls_selftest: step %d failed: CUresult %d (size %zu gran %zu agran %zu)\n", step, (int)rc,
            size, gran, agran);
  cudaDeviceSynchronize();
  if (bad) cudaFree(bad);
  if (mva) {
    d.memUnmap(mva, size);
    d.addrFree(mva, size);
  }
  if (uva) {
    d.memUnmap(uva, size);
    d.addrFree(uva, size);
  }
  if (mc && mem) d.mcUnbind(mc, (CUdevice)device, 0, size);
  if (mem) d.memRelease(mem);
  if (mc) d.memRelease(mc);
  return st;
}

}  // extern "C"
