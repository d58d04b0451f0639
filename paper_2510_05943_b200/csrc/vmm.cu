// vmm.cu -- virtual-memory windows and NVLS multicast teams (NEXT-3 of SURVEY.md §8(f)).
//
// With EARL_NVLS=1 a multi-process comm allocates its window with cuMemCreate instead of
// cudaMalloc, exports it as a POSIX file descriptor (peers fetch the descriptor with
// pidfd_getfd: no socket, no fork), and can bind it to NVSwitch multicast objects: a store to a
// team's multicast address (multimem.st) reaches every member's window at the same offset, so a
// source writes a TP-replicated record once instead of once per replica (egress / R).
//
// The driver entry points come from cudaGetDriverEntryPoint: the library has no link-time
// dependency on libcuda (it still loads on a machine without a driver, for the ABI tests).
#include <cuda.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cstring>

#include "earl_internal.cuh"

namespace earl {

namespace {

struct DriverApi {
  bool ok = false;
  CUresult (*cuDeviceGet)(CUdevice*, int) = nullptr;
  CUresult (*cuMemGetAllocationGranularity)(size_t*, const CUmemAllocationProp*,
                                            CUmemAllocationGranularity_flags) = nullptr;
  CUresult (*cuMemCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*,
                          unsigned long long) = nullptr;
  CUresult (*cuMemRelease)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*cuMemAddressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*cuMemAddressFree)(CUdeviceptr, size_t) = nullptr;
  CUresult (*cuMemMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*cuMemUnmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*cuMemSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  CUresult (*cuMemExportToShareableHandle)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType,
                                           unsigned long long) = nullptr;
  CUresult (*cuMemImportFromShareableHandle)(CUmemGenericAllocationHandle*, void*,
                                             CUmemAllocationHandleType) = nullptr;
  CUresult (*cuMulticastCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*) = nullptr;
  CUresult (*cuMulticastAddDevice)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
  CUresult (*cuMulticastBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle,
                                 size_t, size_t, unsigned long long) = nullptr;
  CUresult (*cuMulticastUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
  CUresult (*cuMulticastGetGranularity)(size_t*, const CUmulticastObjectProp*,
                                        CUmulticastGranularity_flags) = nullptr;
  CUresult (*cuGetErrorString)(CUresult, const char**) = nullptr;
};

template <class F>
bool entry(const char* name, F*& fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || !p) {
    cudaGetLastError();
    return false;
  }
  fn = reinterpret_cast<F*>(p);
  return true;
}

const DriverApi& api() {
  static DriverApi d = [] {
    DriverApi x;
    x.ok = entry("cuDeviceGet", x.cuDeviceGet) &&
           entry("cuMemGetAllocationGranularity", x.cuMemGetAllocationGranularity) &&
           entry("cuMemCreate", x.cuMemCreate) && entry("cuMemRelease", x.cuMemRelease) &&
           entry("cuMemAddressReserve", x.cuMemAddressReserve) &&
           entry("cuMemAddressFree", x.cuMemAddressFree) && entry("cuMemMap", x.cuMemMap) &&
           entry("cuMemUnmap", x.cuMemUnmap) && entry("cuMemSetAccess", x.cuMemSetAccess) &&
           entry("cuMemExportToShareableHandle", x.cuMemExportToShareableHandle) &&
           entry("cuMemImportFromShareableHandle", x.cuMemImportFromShareableHandle) &&
           entry("cuGetErrorString", x.cuGetErrorString);
    // multicast is optional (older drivers): checked again where it is used
    entry("cuMulticastCreate", x.cuMulticastCreate);
    entry("cuMulticastAddDevice", x.cuMulticastAddDevice);
    entry("cuMulticastBindMem", x.cuMulticastBindMem);
    entry("cuMulticastUnbind", x.cuMulticastUnbind);
    entry("cuMulticastGetGranularity", x.cuMulticastGetGranularity);
    return x;
  }();
  return d;
}

const char* cu_err(CUresult r) {
  const char* s = nullptr;
  if (api().cuGetErrorString) api().cuGetErrorString(r, &s);
  return s ? s : "unknown driver error";
}

CUmemAccessDesc rw_access(int device) {
  CUmemAccessDesc acc;
  std::memset(&acc, 0, sizeof(acc));
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  return acc;
}

// reserve + map + grant this device read/write
bool map_handle(CUmemGenericAllocationHandle h, size_t size, int device, uint64_t* va, const char** why) {
  const DriverApi& d = api();
  CUdeviceptr p = 0;
  CUresult r = d.cuMemAddressReserve(&p, size, 0, 0, 0);
  if (r == CUDA_SUCCESS) r = d.cuMemMap(p, size, 0, h, 0);
  if (r == CUDA_SUCCESS) {
    const CUmemAccessDesc acc = rw_access(device);
    r = d.cuMemSetAccess(p, size, &acc, 1);
  }
  if (r != CUDA_SUCCESS) {
    if (p) { d.cuMemUnmap(p, size); d.cuMemAddressFree(p, size); }
    *why = cu_err(r);
    return false;
  }
  *va = (uint64_t)p;
  return true;
}

// A descriptor of process `pid` as a descriptor of this process (Linux >= 5.6; same user).
int fetch_fd(int32_t pid, int32_t fd) {
  const int pfd = (int)syscall(SYS_pidfd_open, (pid_t)pid, 0);
  if (pfd < 0) return -1;
  const int got = (int)syscall(SYS_pidfd_getfd, pfd, fd, 0);
  close(pfd);
  return got;
}

}  // namespace

bool vmm_available() { return api().ok; }
bool multicast_entry_points() {
  const DriverApi& d = api();
  return d.ok && d.cuMulticastCreate && d.cuMulticastAddDevice && d.cuMulticastBindMem &&
         d.cuMulticastGetGranularity;
}

bool vmm_create(int device, uint64_t bytes, VmmMem* out, const char** why) {
  const DriverApi& d = api();
  if (!d.ok) { *why = "driver VMM entry points unavailable"; return false; }
  CUmemAllocationProp prop;
  std::memset(&prop, 0, sizeof(prop));
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = device;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  CUresult r = d.cuMemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
  if (r != CUDA_SUCCESS) { *why = cu_err(r); return false; }
  // a multiple of the multicast granularity too, so the whole window can be bound to a team
  size_t mgran = 0;
  if (multicast_entry_points()) {
    CUmulticastObjectProp mp;
    std::memset(&mp, 0, sizeof(mp));
    mp.numDevices = 1;
    mp.size = gran;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    if (d.cuMulticastGetGranularity(&mgran, &mp, CU_MULTICAST_GRANULARITY_MINIMUM) != CUDA_SUCCESS) mgran = 0;
  }
  if (mgran > gran && mgran % gran == 0) gran = mgran;
  const uint64_t size = (bytes + gran - 1) / gran * gran;
  CUmemGenericAllocationHandle h = 0;
  r = d.cuMemCreate(&h, size, &prop, 0);
  if (r != CUDA_SUCCESS) { *why = cu_err(r); return false; }
  uint64_t va = 0;
  if (!map_handle(h, size, device, &va, why)) { d.cuMemRelease(h); return false; }
  out->handle = (uint64_t)h;
  out->va = va;
  out->size = size;
  out->fd = -1;
  return true;
}

bool vmm_export(VmmMem* m, int32_t* fd, const char** why) {
  const DriverApi& d = api();
  if (m->fd < 0) {
    int f = -1;
    const CUresult r = d.cuMemExportToShareableHandle(&f, (CUmemGenericAllocationHandle)m->handle,
                                                      CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
    if (r != CUDA_SUCCESS) { *why = cu_err(r); return false; }
    m->fd = f;
  }
  *fd = m->fd;
  return true;
}

bool vmm_import(int device, int32_t pid, int32_t fd, uint64_t size, VmmMem* out, const char** why) {
  const DriverApi& d = api();
  if (!d.ok) { *why = "driver VMM entry points unavailable"; return false; }
  const int local = fetch_fd(pid, fd);
  if (local < 0) { *why = "pidfd_getfd failed (kernel < 5.6 or ptrace not permitted)"; return false; }
  CUmemGenericAllocationHandle h = 0;
  const CUresult r = d.cuMemImportFromShareableHandle(&h, (void*)(intptr_t)local,
                                                      CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
  close(local);
  if (r != CUDA_SUCCESS) { *why = cu_err(r); return false; }
  uint64_t va = 0;
  if (!map_handle(h, size, device, &va, why)) { d.cuMemRelease(h); return false; }
  out->handle = (uint64_t)h;
  out->va = va;
  out->size = size;
  out->fd = -1;
  return true;
}

void vmm_free(VmmMem* m) {
  const DriverApi& d = api();
  if (!d.ok || !m->size) return;
  if (m->va) { d.cuMemUnmap((CUdeviceptr)m->va, m->size); d.cuMemAddressFree((CUdeviceptr)m->va, m->size); }
  if (m->handle) d.cuMemRelease((CUmemGenericAllocationHandle)m->handle);
  if (m->fd >= 0) close(m->fd);
  std::memset(m, 0, sizeof(*m));
  m->fd = -1;
}

bool mc_create(int n_devices, uint64_t size, VmmMem* out, const char** why) {
  const DriverApi& d = api();
  if (!multicast_entry_points()) { *why = "driver has no multicast entry points"; return false; }
  CUmulticastObjectProp mp;
  std::memset(&mp, 0, sizeof(mp));
  mp.numDevices = (unsigned)n_devices;
  mp.size = size;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  CUmemGenericAllocationHandle h = 0;
  const CUresult r = d.cuMulticastCreate(&h, &mp);
  if (r != CUDA_SUCCESS) { *why = cu_err(r); return false; }
  out->handle = (uint64_t)h;
  out->va = 0;
  out->size = size;
  out->fd = -1;
  return true;
}

bool mc_import(int32_t pid, int32_t fd, uint64_t size, VmmMem* out, const char** why) {
  const DriverApi& d = api();
  const int local = fetch_fd(pid, fd);
  if (local < 0) { *why = "pidfd_getfd failed"; return false; }
  CUmemGenericAllocationHandle h = 0;
  const CUresult r = d.cuMemImportFromShareableHandle(&h, (void*)(intptr_t)local,
                                                      CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
  close(local);
  if (r != CUDA_SUCCESS) { *why = cu_err(r); return false; }
  out->handle = (uint64_t)h;
  out->va = 0;
  out->size = size;
  out->fd = -1;
  return true;
}

// Add this device to the team, bind the window to it at offset 0, map the multicast address.
// cuMulticastBindMem blocks until every member has added its device: every member calls this
// concurrently (collective).
bool mc_join(VmmMem* mc, int device, const VmmMem& window, const char** why) {
  const DriverApi& d = api();
  CUdevice dev = 0;
  CUresult r = d.cuDeviceGet(&dev, device);
  if (r == CUDA_SUCCESS) r = d.cuMulticastAddDevice((CUmemGenericAllocationHandle)mc->handle, dev);
  if (r == CUDA_SUCCESS)
    r = d.cuMulticastBindMem((CUmemGenericAllocationHandle)mc->handle, 0,
                             (CUmemGenericAllocationHandle)window.handle, 0, mc->size, 0);
  if (r != CUDA_SUCCESS) { *why = cu_err(r); return false; }
  uint64_t va = 0;
  if (!map_handle((CUmemGenericAllocationHandle)mc->handle, mc->size, device, &va, why)) return false;
  mc->va = va;
  return true;
}

void mc_free(VmmMem* mc, int device) {
  const DriverApi& d = api();
  if (!mc->handle) return;
  if (mc->va) { d.cuMemUnmap((CUdeviceptr)mc->va, mc->size); d.cuMemAddressFree((CUdeviceptr)mc->va, mc->size); }
  CUdevice dev = 0;
  if (d.cuMulticastUnbind && d.cuDeviceGet(&dev, device) == CUDA_SUCCESS)
    d.cuMulticastUnbind((CUmemGenericAllocationHandle)mc->handle, dev, 0, mc->size);
  d.cuMemRelease((CUmemGenericAllocationHandle)mc->handle);
  if (mc->fd >= 0) close(mc->fd);
  std::memset(mc, 0, sizeof(*mc));
  mc->fd = -1;
}

}  // namespace earl
