// nvls_probe.cu -- what the B200 box supports for NEXT-3 (NVLS multicast), before building it:
//   * CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, handle types, granularities
//   * a 1-device multicast object: create, add device, bind a cuMemCreate allocation, map the
//     multicast VA, multimem.st from a kernel, read back through the unicast VA
//   * POSIX-FD export of a cuMemCreate allocation and pidfd_getfd in a forked child (the FD
//     passing a multi-process window / multicast setup needs)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o nvls_probe nvls_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <errno.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/syscall.h>
#include <sys/wait.h>
#include <unistd.h>

#define CK(x)                                                                          \
  do {                                                                                 \
    CUresult r_ = (x);                                                                 \
    if (r_ != CUDA_SUCCESS) {                                                          \
      const char* s_ = nullptr;                                                        \
      cuGetErrorString(r_, &s_);                                                       \
      printf("FAIL %s -> %d %s\n", #x, (int)r_, s_ ? s_ : "?");                        \
      return 1;                                                                        \
    }                                                                                  \
  } while (0)

__global__ void mc_store(float* mc, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (4 * i + 3 < n) {
    float4 v = make_float4(4 * i, 4 * i + 1, 4 * i + 2, 4 * i + 3);
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + 4 * i),
                 "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
  }
}

int main() {
  CK(cuInit(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  CUcontext ctx;
  CK(cuDevicePrimaryCtxRetain(&ctx, dev));
  CK(cuCtxSetCurrent(ctx));
  int mc = 0, fabric = 0, posix = 0, vmm = 0;
  CK(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  CK(cuDeviceGetAttribute(&vmm, CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED, dev));
  CK(cuDeviceGetAttribute(&posix, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED, dev));
  cuDeviceGetAttribute(&fabric, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
  printf("multicast_supported=%d vmm=%d posix_fd=%d fabric=%d\n", mc, vmm, posix, fabric);

  // a cuMemCreate allocation, exportable as a POSIX FD
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = 0;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  CK(cuMemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  const size_t size = 32 * gran;
  printf("mem granularity=%zu size=%zu\n", gran, size);
  CUmemGenericAllocationHandle mem;
  CK(cuMemCreate(&mem, size, &prop, 0));
  CUdeviceptr uva;
  CK(cuMemAddressReserve(&uva, size, 0, 0, 0));
  CK(cuMemMap(uva, size, 0, mem, 0));
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = 0;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(uva, size, &acc, 1));
  CK(cuMemsetD8(uva, 0, size));

  // FD export + pidfd_getfd from a child process
  int fd = -1;
  CK(cuMemExportToShareableHandle(&fd, mem, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
  printf("exported fd=%d\n", fd);
  pid_t parent = getpid();
  pid_t ch = fork();
  if (ch == 0) {
    int pfd = (int)syscall(SYS_pidfd_open, parent, 0);
    int got = pfd >= 0 ? (int)syscall(SYS_pidfd_getfd, pfd, fd, 0) : -1;
    printf("child: pidfd_open=%d pidfd_getfd=%d (%s)\n", pfd, got, got < 0 ? strerror(errno) : "ok");
    _exit(got >= 0 ? 0 : 3);
  }
  int st = 0;
  waitpid(ch, &st, 0);
  printf("pidfd_getfd in child: %s\n", WIFEXITED(st) && WEXITSTATUS(st) == 0 ? "works" : "FAILS");

  if (!mc) { printf("no multicast: stop\n"); return 0; }
  CUmulticastObjectProp mp = {};
  mp.numDevices = 1;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t mgran = 0, mrec = 0;
  mp.size = size;
  CK(cuMulticastGetGranularity(&mgran, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
  CK(cuMulticastGetGranularity(&mrec, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  printf("multicast granularity min=%zu recommended=%zu\n", mgran, mrec);
  CUmemGenericAllocationHandle mch;
  // which properties does this box accept? (size: min vs recommended granularity; handle
  // types: POSIX FD, fabric, none)
  CUresult cr = CUDA_ERROR_INVALID_VALUE;
  const unsigned long long htypes[3] = {CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
                                        CU_MEM_HANDLE_TYPE_FABRIC, 0};
  const size_t sizes[2] = {((size + mgran - 1) / mgran) * mgran, ((size + mrec - 1) / mrec) * mrec};
  for (int hi = 0; hi < 3 && cr != CUDA_SUCCESS; ++hi)
    for (int si = 0; si < 2 && cr != CUDA_SUCCESS; ++si) {
      mp.handleTypes = htypes[hi];
      mp.size = sizes[si];
      cr = cuMulticastCreate(&mch, &mp);
      const char* es = nullptr;
      cuGetErrorString(cr, &es);
      printf("cuMulticastCreate(numDevices=1, handleTypes=0x%llx, size=%zu) -> %d %s\n",
             htypes[hi], sizes[si], (int)cr, es ? es : "?");
    }
  if (cr != CUDA_SUCCESS) {
    mp.numDevices = 2;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    mp.size = sizes[0];
    cr = cuMulticastCreate(&mch, &mp);
    printf("cuMulticastCreate(numDevices=2) -> %d\n", (int)cr);
    return 0;
  }
  CK(cuMulticastAddDevice(mch, dev));
  CK(cuMulticastBindMem(mch, 0, mem, 0, size, 0));
  CUdeviceptr mcva;
  CK(cuMemAddressReserve(&mcva, mp.size, 0, 0, 0));
  CK(cuMemMap(mcva, mp.size, 0, mch, 0));
  CK(cuMemSetAccess(mcva, mp.size, &acc, 1));
  const int n = 1 << 20;
  mc_store<<<n / 4 / 256, 256>>>((float*)mcva, n);
  cudaError_t e = cudaDeviceSynchronize();
  printf("multimem.st kernel: %s\n", cudaGetErrorString(e));
  float* h = (float*)malloc(n * 4);
  CK(cuMemcpyDtoH(h, uva, n * 4));
  int bad = 0;
  for (int i = 0; i < n; ++i) bad += h[i] != (float)i;
  printf("multicast write visible through the unicast mapping: %s (%d bad)\n", bad ? "NO" : "yes", bad);
  return 0;
}
