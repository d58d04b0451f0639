// lengths.cu -- step a1 of SURVEY.md §8(a): the global length vector on every rank, gathered on
// the device (the layout knowledge the dispatcher plans from, "using the selected parallelism
// and data layout").
//
// Global sequence order is rank-major (reading c6): rank r's counts[r] local lengths occupy
// [sum_{q<r} counts[q], +counts[r]) of the global vector.  The counts are host values fixed by
// the source layout (rollout GIVEN_COUNTS), so the gather is one kernel with no host round trip
// and is capturable into a CUDA graph together with the planner and the exchange.
//
// Multi-process comm: every rank stores its lengths into every peer's gather area (a double
// buffer after the signal pad of each window, selected by the gather epoch's parity) with 16-B
// stores over NVLink, releases the epoch into each peer's pad, acquires every peer's, and copies
// the completed area into the caller's output.  The double buffer is safe without a second
// barrier: a peer can write gather e+2 into this rank's area only after this rank's gather e+1
// signalled, which is stream-ordered after gather e's copy-out.
#include "earl_internal.cuh"

namespace earl {

namespace {

constexpr int kThreads = 1024;
constexpr unsigned kFullMask = 0xffffffffu;

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Copy n int32 from src to dst (any alignment of the element index; 16-B vectors where both
// sides allow it), threads [tid0, tid0 + nthreads).
// L2_ONLY: the source was written by peers (loads bypass L1).
template <bool L2_ONLY>
__device__ void copy_i32(int32_t* dst, const int32_t* src, int64_t n, int64_t tid, int64_t nthreads) {
  const bool vec = (((uintptr_t)dst | (uintptr_t)src) & 15) == 0;
  int64_t done = 0;
  if (vec) {
    const int64_t nv = n >> 2;
    const int4* s4 = reinterpret_cast<const int4*>(src);
    for (int64_t k = tid; k < nv; k += nthreads)
      reinterpret_cast<int4*>(dst)[k] = L2_ONLY ? __ldcg(s4 + k) : s4[k];
    done = nv << 2;
  }
  for (int64_t k = done + tid; k < n; k += nthreads) dst[k] = L2_ONLY ? __ldcg(src + k) : src[k];
}

// Multi-process gather: grid of G CTAs stores this rank's lengths into every peer's area; the
// last CTA to finish signals, waits, and copies the area out.
__global__ void __launch_bounds__(kThreads) gather_lengths_kernel(const __grid_constant__ LensArgs a) {
  __shared__ unsigned s_last;
  __shared__ uint64_t s_epoch;
  if (threadIdx.x == 0) s_epoch = *reinterpret_cast<volatile uint64_t*>(a.my_pad + kLensEpochSlot) + 1;
  __syncthreads();
  const uint64_t epoch = s_epoch;
  const int par = (int)(epoch & 1);
  const int64_t mine = a.counts[a.me];
  const int64_t off = a.start[a.me];
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  for (int p = 0; p < a.world; ++p) {
    int32_t* area = reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(a.peer_pad[p]) + kPadBytes) +
                    (int64_t)par * a.cap;
    copy_i32<false>(area + off, a.local, mine, tid, nth);
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(a.ctr, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    if (lane == 0) {
      *a.ctr = 0;
      a.my_pad[kLensEpochSlot] = epoch;
    }
    delay_inject(7);
    __threadfence_system();
    if (lane < a.world && lane != a.me) st_release_sys_u64(a.peer_pad[lane] + kLensSlot + a.me, epoch);
    unsigned missing = 0;
    if (lane < a.world && lane != a.me) {
      const uint64_t t0 = gtimer();
      while (ld_acquire_sys_u64(a.my_pad + kLensSlot + lane) < epoch) {
        if (gtimer() - t0 > a.timeout_ns) { missing = 1u << lane; break; }
        __nanosleep(64);
      }
    }
    missing = __reduce_or_sync(kFullMask, missing);
    if (lane == 0 && missing) {
      if (atomicCAS(a.err, 0, EARL_ERR_TIMEOUT) == 0) a.err[1] = (int32_t)missing;
    }
  }
  __syncthreads();
  __threadfence_system();
  const int32_t* area = reinterpret_cast<const int32_t*>(reinterpret_cast<const uint8_t*>(a.my_pad) + kPadBytes) +
                        (int64_t)par * a.cap;
  copy_i32<true>(a.out, area, a.total, threadIdx.x, blockDim.x);
}

// Emulated comm: the gather is a concatenation of the ranks' local vectors.
__global__ void __launch_bounds__(kThreads) concat_lengths_kernel(const __grid_constant__ LensArgs a) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  for (int r = 0; r < a.world; ++r)
    if (a.counts[r] > 0) copy_i32<false>(a.out + a.start[r], a.src[r], a.counts[r], tid, nth);
}

__global__ void fill_i32_kernel(int32_t* p, int32_t v, int64_t n) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    p[k] = v;
}

}  // namespace

cudaError_t launch_fill_i32(int32_t* p, int32_t v, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  int64_t g = (n + 255) / 256;
  if (g > 1024) g = 1024;
  fill_i32_kernel<<<(int)g, 256, 0, s>>>(p, v, n);
  return cudaGetLastError();
}

cudaError_t launch_gather_lengths(const LensArgs& a, int sm_count, cudaStream_t s) {
  const int64_t per = a.emulated ? a.total : a.counts[a.me] * a.world;
  int64_t g = (per / 4 + kThreads - 1) / kThreads;
  if (g < 1) g = 1;
  if (g > sm_count) g = sm_count;
  if (a.emulated)
    concat_lengths_kernel<<<(int)g, kThreads, 0, s>>>(a);
  else
    gather_lengths_kernel<<<(int)g, kThreads, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace earl
