// api.cu -- host side of libearl_dispatch.so: the C ABI of include/earl_dispatch.h.
//
// Owns argument validation (SURVEY.md §8(b) error list), the comm (symmetric receive windows,
// CUDA-IPC peer mappings, signal pads), plan lifetime (stream-ordered allocations from the
// device memory pool, so a steady-state plan allocates nothing from the driver), and the
// launches of the planner (planner.cu) and the copy kernels (copy.cu).
#include <unistd.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include "earl_internal.cuh"

using namespace earl;

namespace {

thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};

// NVTX range around a C-ABI call that enqueues device work (SURVEY.md §5 tracing): tools (nsys,
// ncu --nvtx --nvtx-include "earl_dispatch_exec/") attribute the kernels to the call; without a
// tool attached the header-only NVTX3 calls are a null-pointer check.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

earl_status_t fail(earl_status_t st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = std::string(earl_status_string(st)) + ": " + buf;
  return st;
}

}  // namespace

namespace earl {
// the last-error slot shared with selector.cpp (host-only code in another translation unit)
earl_status_t set_error(earl_status_t st, const char* msg) { return fail(st, "%s", msg); }
}  // namespace earl

namespace {

#define CUDA_TRY(expr)                                                                     \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return fail(EARL_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_),   \
                  __FILE__, __LINE__);                                                     \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev && cudaSetDevice(dev) != cudaSuccess) cudaGetLastError();
  }
  ~DeviceGuard() {
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess) cur = -1;
    if (prev >= 0 && cur != prev && cudaSetDevice(prev) != cudaSuccess) cudaGetLastError();
  }
};

// Launch checks read cudaGetLastError(); clear any stale error left by an unrelated earlier
// runtime call first, so a launch is never blamed for someone else's failure.
inline void clear_stale_error() { (void)cudaGetLastError(); }

inline bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

}  // namespace

struct earl_comm {
  int32_t rank = 0;      // EARL_ALL_RANKS when emulated
  int32_t world = 1;
  int32_t device = 0;
  bool emulated = false;
  uint64_t window_bytes = 0;
  uint64_t pad_bytes = kPadBytes;  // signal pad + (multi-process) the a1 gather double buffer
  int64_t lens_cap = 0;            // sequences per gather buffer
  uint8_t* win[kMaxWorld] = {};    // local windows (emulated: one per rank; else win[rank])
  uint8_t* peer[kMaxWorld] = {};   // every rank's window as addressable from this process
  bool peer_mapped[kMaxWorld] = {};
  bool peers_ready = false;
  uint64_t alloc_off[kMaxWorld] = {};
  uint64_t epoch = 0;
  unsigned int* done_ctr = nullptr;
  unsigned int* lens_ctr = nullptr;  // a1 gather: last-CTA counter
  int32_t* dev_err = nullptr;        // a1 gather: [status, missing-peer mask] latched on the device
  int sm_count = 148;
  uint64_t timeout_ns = 10ull * 1000 * 1000 * 1000;
  int refs = 1;          // the user's handle + one per live plan: freed when it reaches 0
  // K8, the staged exchange's NCCL comm (earl_comm_init_nccl) and its stage buffers (send,
  // receive), grown on demand; registered with the comm when EARL_NCCL_REGISTER=1
  ncclComm_t nccl = nullptr;
  bool nccl_register = false;
  void* nst[2] = {};
  uint64_t nst_bytes[2] = {};
  void* nreg[2] = {};
  // NEXT-3 (EARL_NVLS=1): the window from cuMemCreate, peers imported by file descriptor, and
  // the multicast teams this rank belongs to (each bound to the whole window at offset 0)
  int32_t node_size = 0;   // NEXT-4: ranks per node (0: the whole comm is one node)
  int32_t opt_remote_tma = -1;  // earl_comm_set_exec_options (-1: the environment's choice)
  int32_t opt_p2p_shape = -1;
  bool vmm = false;
  VmmMem vwin{0, 0, 0, -1};
  VmmMem vpeer[kMaxWorld] = {};
  struct Team {
    uint32_t mask;
    VmmMem mc;
  } teams[kMaxShards] = {};
  int n_teams = 0;
};

namespace {
// NEXT-4: the node of a rank, and the ranks of this rank's node
inline int node_of(const earl_comm* c, int r) { return c->node_size > 0 ? r / c->node_size : 0; }
inline bool same_node(const earl_comm* c, int a, int b) { return node_of(c, a) == node_of(c, b); }
inline uint32_t node_mask(const earl_comm* c) {
  uint32_t m = 0;
  for (int p = 0; p < c->world; ++p)
    if (c->emulated || same_node(c, p, c->rank)) m |= 1u << p;
  return m;
}
constexpr uint32_t kVmmMagic = 0x4d4d5645u;   // "EVMM": a cuMemCreate window handle
constexpr uint32_t kTeamMagic = 0x544d4345u;  // "ECMT": a multicast team handle
struct FdHandle {
  uint32_t magic;
  int32_t pid;
  int32_t fd;
  int32_t pad;
  uint64_t size;
  uint32_t mask;
};
static_assert(sizeof(FdHandle) <= EARL_HANDLE_BYTES, "handle size");
}  // namespace

namespace {
void comm_release(earl_comm* c) {
  if (--c->refs > 0) return;
  DeviceGuard g(c->device);
  cudaDeviceSynchronize();
  for (int t = 0; t < kMaxShards; ++t)  // joined teams, and a created one not joined yet
    if (c->teams[t].mc.handle) mc_free(&c->teams[t].mc, c->device);
  for (int p = 0; p < kMaxWorld; ++p) {
    if (!c->peer_mapped[p]) continue;
    if (c->vmm) vmm_free(&c->vpeer[p]);
    else cudaIpcCloseMemHandle(c->peer[p]);
  }
  if (c->vmm) {
    vmm_free(&c->vwin);
  } else {
    for (int r = 0; r < kMaxWorld; ++r)
      if (c->win[r]) cudaFree(c->win[r]);
  }
  for (int k = 0; k < 2; ++k) {
    if (c->nreg[k]) ncclCommDeregister(c->nccl, c->nreg[k]);
    if (c->nst[k]) {
      if (c->nccl_register) ncclMemFree(c->nst[k]);
      else cudaFree(c->nst[k]);
    }
  }
  if (c->nccl) ncclCommDestroy(c->nccl);
  if (c->done_ctr) cudaFree(c->done_ctr);
  if (c->lens_ctr) cudaFree(c->lens_ctr);
  if (c->dev_err) cudaFree(c->dev_err);
  cudaGetLastError();
  delete c;
}
}  // namespace

struct earl_plan {
  earl_comm* comm = nullptr;
  PlanArgs args{};
  earl_layout_t lay[2]{};
  int64_t N = 0;
  int32_t n_fields = 0;
  earl_field_t fields[kMaxFields]{};
  void* mem = nullptr;
  size_t mem_bytes = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev = nullptr;   // recorded after the plan's last launch (use_end)
  bool ev_recorded = false;
  bool synced = false;
  PlanHeader host_hdr{};
  size_t lpt_smem = 0;
  int grid = 1;
  void* agg_ws = nullptr;     // returns_kernel look-back workspace (AggWork + AggWindow[agg_cap])
  int64_t agg_cap = 0;
  // per-sequence field plan (earl_plan_seq_fields): the token plan it follows (referenced, so it
  // outlives this plan) and this plan's own device arrays [g_src | g_dst | ones], N int32 each
  earl_plan* parent = nullptr;
  int32_t* owned = nullptr;
  int refs = 1;
  bool fast = false;          // the SP = 1 single-pass planner (planner_sp1_kernel)
};

// ---------------------------------------------------------------------------------------
// misc
// ---------------------------------------------------------------------------------------

extern "C" const char* earl_status_string(earl_status_t st) {
  switch (st) {
    case EARL_OK: return "EARL_OK";
    case EARL_ERR_INVALID_ARGUMENT: return "EARL_ERR_INVALID_ARGUMENT";
    case EARL_ERR_LAYOUT: return "EARL_ERR_LAYOUT";
    case EARL_ERR_CAPACITY: return "EARL_ERR_CAPACITY";
    case EARL_ERR_CUDA: return "EARL_ERR_CUDA";
    case EARL_ERR_NCCL: return "EARL_ERR_NCCL";
    case EARL_ERR_TIMEOUT: return "EARL_ERR_TIMEOUT";
    case EARL_ERR_MISMATCH: return "EARL_ERR_MISMATCH";
    case EARL_ERR_UNSUPPORTED: return "EARL_ERR_UNSUPPORTED";
    case EARL_ERR_POLICY: return "EARL_ERR_POLICY";
  }
  return "EARL_ERR_UNKNOWN";
}

extern "C" const char* earl_last_error(void) { return g_last_error.c_str(); }
extern "C" int32_t earl_abi_version(void) { return EARL_ABI_VERSION; }
extern "C" uint64_t earl_kernel_launch_count(void) { return g_launches.load(); }

// ---------------------------------------------------------------------------------------
// comm
// ---------------------------------------------------------------------------------------

extern "C" earl_status_t earl_comm_create(int32_t rank, int32_t world, int32_t cuda_device,
                                          uint64_t window_bytes, earl_comm_t* out) {
  if (!out) return fail(EARL_ERR_INVALID_ARGUMENT, "comm out-pointer is NULL");
  *out = nullptr;
  if (world < 1 || world > kMaxWorld)
    return fail(EARL_ERR_UNSUPPORTED, "world %d outside [1, %d]", world, kMaxWorld);
  if (rank != EARL_ALL_RANKS && (rank < 0 || rank >= world))
    return fail(EARL_ERR_INVALID_ARGUMENT, "rank %d outside [0, %d)", rank, world);
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (cuda_device < 0 || cuda_device >= ndev)
    return fail(EARL_ERR_INVALID_ARGUMENT, "cuda_device %d outside [0, %d)", cuda_device, ndev);
  DeviceGuard g(cuda_device);
  earl_comm* c = new earl_comm();
  c->rank = rank;
  c->world = world;
  c->device = cuda_device;
  c->emulated = (rank == EARL_ALL_RANKS);
  // multi-process windows carry the a1 gather area after the signal pad: 2 x lens_cap int32
  // (EARL_LENS_CAPACITY sequences, default 2^18 = 2 MiB per window)
  if (!c->emulated && world > 1) {
    c->lens_cap = int64_t(1) << 18;
    if (const char* lc = getenv("EARL_LENS_CAPACITY")) {
      const long long v = atoll(lc);
      if (v > 0) c->lens_cap = (v + 3) & ~3LL;
    }
    c->pad_bytes = kPadBytes + (((uint64_t)c->lens_cap * 8 + 255) & ~255ull);
  }
  c->window_bytes = ((window_bytes + 255) & ~255ull) + c->pad_bytes;
  if (const char* t = getenv("EARL_TIMEOUT_MS")) {  // peer waits (SPEC.md:316 barrier timeout)
    const long long ms = atoll(t);
    if (ms > 0) c->timeout_ns = (uint64_t)ms * 1000000ull;
  }
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, cuda_device);
  // keep freed plan memory cached in the pool: steady-state planning never calls the driver
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, cuda_device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  auto cleanup = [&](earl_status_t st) {
    earl_comm_destroy(c);
    return st;
  };
  const int nwin = c->emulated ? world : 1;
  const char* nvls = getenv("EARL_NVLS");
  c->vmm = !c->emulated && world > 1 && nvls && atoi(nvls) != 0;
  for (int r = 0; r < nwin; ++r) {
    const int rr = c->emulated ? r : rank;
    if (c->vmm) {  // NEXT-3: a cuMemCreate window (bindable to multicast teams)
      const char* why = "";
      if (!vmm_create(cuda_device, c->window_bytes, &c->vwin, &why))
        return cleanup(fail(EARL_ERR_UNSUPPORTED, "EARL_NVLS=1: cuMemCreate window: %s", why));
      c->window_bytes = c->vwin.size;
      c->win[rr] = reinterpret_cast<uint8_t*>(c->vwin.va);
      cudaError_t e = cudaMemset(c->win[rr], 0, kPadBytes);
      if (e != cudaSuccess) return cleanup(fail(EARL_ERR_CUDA, "pad memset: %s", cudaGetErrorString(e)));
      c->peer[rr] = c->win[rr];
      c->alloc_off[rr] = c->pad_bytes;
      continue;
    }
    cudaError_t e = cudaMalloc(&c->win[rr], c->window_bytes);
    if (e != cudaSuccess)
      return cleanup(fail(EARL_ERR_CUDA, "window cudaMalloc(%llu): %s",
                          (unsigned long long)c->window_bytes, cudaGetErrorString(e)));
    e = cudaMemset(c->win[rr], 0, kPadBytes);
    if (e != cudaSuccess) return cleanup(fail(EARL_ERR_CUDA, "pad memset: %s", cudaGetErrorString(e)));
    c->peer[rr] = c->win[rr];
    c->alloc_off[rr] = c->pad_bytes;
  }
  cudaError_t e = cudaMalloc(&c->done_ctr, sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaMemset(c->done_ctr, 0, sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaMalloc(&c->lens_ctr, sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaMemset(c->lens_ctr, 0, sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaMalloc(&c->dev_err, 2 * sizeof(int32_t));
  if (e == cudaSuccess) e = cudaMemset(c->dev_err, 0, 2 * sizeof(int32_t));
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cleanup(fail(EARL_ERR_CUDA, "comm init: %s", cudaGetErrorString(e)));
  c->peers_ready = c->emulated || world == 1;
  *out = c;
  return EARL_OK;
}

extern "C" earl_status_t earl_comm_export_handle(earl_comm_t c, void* handle_out) {
  if (!c || !handle_out) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL argument");
  if (c->emulated) return fail(EARL_ERR_UNSUPPORTED, "emulated comm has no peers to export to");
  static_assert(sizeof(cudaIpcMemHandle_t) <= EARL_HANDLE_BYTES, "handle size");
  DeviceGuard g(c->device);
  std::memset(handle_out, 0, EARL_HANDLE_BYTES);
  if (c->vmm) {
    FdHandle fh{};
    const char* why = "";
    if (!vmm_export(&c->vwin, &fh.fd, &why))
      return fail(EARL_ERR_CUDA, "window export: %s", why);
    fh.magic = kVmmMagic;
    fh.pid = (int32_t)getpid();
    fh.size = c->vwin.size;
    std::memcpy(handle_out, &fh, sizeof(fh));
    return EARL_OK;
  }
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, c->win[c->rank]));
  std::memcpy(handle_out, &h, sizeof(h));
  return EARL_OK;
}

extern "C" earl_status_t earl_comm_import_peers(earl_comm_t c, const void* handles) {
  if (!c || !handles) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL argument");
  if (c->emulated) return fail(EARL_ERR_UNSUPPORTED, "emulated comm has no peers to import");
  DeviceGuard g(c->device);
  const uint8_t* hb = static_cast<const uint8_t*>(handles);
  for (int p = 0; p < c->world; ++p) {
    if (p == c->rank || c->peer_mapped[p]) continue;
    if (!same_node(c, p, c->rank)) continue;  // NEXT-4: other nodes are reached by NCCL only
    FdHandle fh;
    std::memcpy(&fh, hb + (size_t)p * EARL_HANDLE_BYTES, sizeof(fh));
    if ((fh.magic == kVmmMagic) != c->vmm)
      return fail(EARL_ERR_INVALID_ARGUMENT, "peer %d's window kind differs (EARL_NVLS must match on every rank)", p);
    if (c->vmm) {
      const char* why = "";
      if (!vmm_import(c->device, fh.pid, fh.fd, fh.size, &c->vpeer[p], &why))
        return fail(EARL_ERR_CUDA, "import of peer %d's window: %s", p, why);
      c->peer[p] = reinterpret_cast<uint8_t*>(c->vpeer[p].va);
      c->peer_mapped[p] = true;
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, hb + (size_t)p * EARL_HANDLE_BYTES, sizeof(h));
    void* ptr = nullptr;
    CUDA_TRY(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    c->peer[p] = static_cast<uint8_t*>(ptr);
    c->peer_mapped[p] = true;
  }
  c->peers_ready = true;
  return EARL_OK;
}

extern "C" earl_status_t earl_comm_alloc(earl_comm_t c, int32_t rank, uint64_t bytes, void** ptr) {
  if (!c || !ptr) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL argument");
  const int r = c->emulated ? rank : c->rank;
  if (r < 0 || r >= c->world || !c->win[r])
    return fail(EARL_ERR_INVALID_ARGUMENT, "rank %d has no local window", rank);
  const uint64_t need = (bytes + 255) & ~255ull;
  if (c->alloc_off[r] + need > c->window_bytes)
    return fail(EARL_ERR_CAPACITY, "window of rank %d exhausted: %llu + %llu > %llu", r,
                (unsigned long long)c->alloc_off[r], (unsigned long long)need,
                (unsigned long long)c->window_bytes);
  *ptr = c->win[r] + c->alloc_off[r];
  c->alloc_off[r] += need;
  return EARL_OK;
}

extern "C" earl_status_t earl_comm_reset_alloc(earl_comm_t c) {
  if (!c) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL comm");
  for (int r = 0; r < kMaxWorld; ++r) c->alloc_off[r] = c->pad_bytes;
  return EARL_OK;
}

extern "C" earl_status_t earl_comm_info(earl_comm_t c, int32_t* rank, int32_t* world,
                                        int32_t* emulated) {
  if (!c) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL comm");
  if (rank) *rank = c->rank;
  if (world) *world = c->world;
  if (emulated) *emulated = c->emulated ? 1 : 0;
  return EARL_OK;
}

extern "C" earl_status_t earl_allgather_lengths(earl_comm_t c, const int64_t* counts,
                                                const void* const* local_lens, int32_t* global_lens,
                                                void* stream) {
  NvtxRange nvtx("earl_allgather_lengths");
  if (!c || !counts || !local_lens) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL argument");
  if (!c->peers_ready)
    return fail(EARL_ERR_INVALID_ARGUMENT, "multi-process comm: earl_comm_import_peers not called");
  LensArgs a;
  std::memset(&a, 0, sizeof(a));
  a.world = c->world;
  a.emulated = c->emulated ? 1 : 0;
  a.me = c->emulated ? 0 : c->rank;
  int64_t tot = 0;
  for (int r = 0; r < c->world; ++r) {
    if (counts[r] < 0) return fail(EARL_ERR_INVALID_ARGUMENT, "counts[%d] < 0", r);
    a.counts[r] = counts[r];
    a.start[r] = tot;
    tot += counts[r];
  }
  if (tot > 0x7fffffffLL) return fail(EARL_ERR_INVALID_ARGUMENT, "more than 2^31 - 1 sequences");
  a.total = tot;
  if (tot > 0 && !global_lens) return fail(EARL_ERR_INVALID_ARGUMENT, "global_lens is NULL");
  a.out = global_lens;
  if (c->emulated) {
    for (int r = 0; r < c->world; ++r) {
      a.src[r] = static_cast<const int32_t*>(local_lens[r]);
      if (counts[r] > 0 && !a.src[r])
        return fail(EARL_ERR_INVALID_ARGUMENT, "local_lens[%d] is NULL with counts %lld", r,
                    (long long)counts[r]);
    }
  } else {
    a.local = static_cast<const int32_t*>(local_lens[0]);
    if (counts[c->rank] > 0 && !a.local)
      return fail(EARL_ERR_INVALID_ARGUMENT, "local_lens is NULL with counts %lld",
                  (long long)counts[c->rank]);
  }
  DeviceGuard g(c->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  clear_stale_error();
  if (c->node_size > 0)
    return fail(EARL_ERR_UNSUPPORTED,
                "multi-node comm: the device gather reaches one node; gather lengths over the process group");
  if (!c->emulated && c->world == 1) {  // one rank: the global vector is the local one
    if (tot > 0) CUDA_TRY(cudaMemcpyAsync(global_lens, a.local, tot * 4, cudaMemcpyDeviceToDevice, s));
    return EARL_OK;
  }
  if (tot == 0 && c->emulated) return EARL_OK;
  if (!c->emulated) {
    if (tot > c->lens_cap)
      return fail(EARL_ERR_CAPACITY, "%lld sequences exceed the gather capacity %lld (EARL_LENS_CAPACITY)",
                  (long long)tot, (long long)c->lens_cap);
    a.cap = c->lens_cap;
    a.my_pad = reinterpret_cast<uint64_t*>(c->win[c->rank]);
    for (int q = 0; q < c->world; ++q) a.peer_pad[q] = reinterpret_cast<uint64_t*>(c->peer[q]);
    a.ctr = c->lens_ctr;
    a.err = c->dev_err;
    a.timeout_ns = c->timeout_ns;
  }
  cudaError_t e = launch_gather_lengths(a, c->sm_count, s);
  if (e != cudaSuccess) return fail(EARL_ERR_CUDA, "length gather launch: %s", cudaGetErrorString(e));
  g_launches.fetch_add(1);
  return EARL_OK;
}

extern "C" earl_status_t earl_comm_check(earl_comm_t c, void* stream) {
  if (!c) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL comm");
  DeviceGuard g(c->device);
  int32_t h[2] = {0, 0};
  CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  CUDA_TRY(cudaMemcpy(h, c->dev_err, sizeof(h), cudaMemcpyDeviceToHost));
  if (h[0] == 0) return EARL_OK;
  CUDA_TRY(cudaMemset(c->dev_err, 0, sizeof(h)));
  return fail((earl_status_t)h[0], "length gather: peers missing (mask 0x%x)", h[1]);
}

extern "C" earl_status_t earl_comm_set_exec_options(earl_comm_t c, int32_t remote_store,
                                                    int32_t p2p_shape) {
  if (!c) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL comm");
  if (remote_store < -1 || remote_store > 1)
    return fail(EARL_ERR_INVALID_ARGUMENT, "remote_store %d outside {-1, 0, 1}", remote_store);
  static const int shapes[] = {-1, 1, 2, 3, 4, 5, 6, 7, 8, 11, 14};
  bool known = false;
  for (int v : shapes) known |= v == p2p_shape;
  if (!known) return fail(EARL_ERR_INVALID_ARGUMENT, "unknown copy-engine shape %d", p2p_shape);
  c->opt_remote_tma = remote_store;
  c->opt_p2p_shape = p2p_shape;
  return EARL_OK;
}

extern "C" earl_status_t earl_comm_set_nodes(earl_comm_t c, int32_t node_size) {
  if (!c) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL comm");
  if (c->emulated) return fail(EARL_ERR_UNSUPPORTED, "emulated comm: one process holds every rank");
  if (c->peers_ready && c->world > 1)
    return fail(EARL_ERR_INVALID_ARGUMENT, "earl_comm_set_nodes must precede earl_comm_import_peers");
  if (node_size < 1 || c->world % node_size != 0)
    return fail(EARL_ERR_INVALID_ARGUMENT, "node size %d does not divide the world of %d", node_size, c->world);
  c->node_size = node_size >= c->world ? 0 : node_size;
  return EARL_OK;
}

extern "C" earl_status_t earl_comm_peer_mask(earl_comm_t c, uint32_t* mask) {
  if (!c || !mask) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL argument");
  uint32_t m = 0;
  for (int p = 0; p < c->world; ++p)
    if (c->peer_mapped[p]) m |= 1u << p;
  *mask = m;
  return EARL_OK;
}

extern "C" earl_status_t earl_comm_mc_create(earl_comm_t c, uint32_t team_mask, void* handle_out) {
  if (!c || !handle_out) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL argument");
  if (!c->vmm) return fail(EARL_ERR_UNSUPPORTED, "multicast teams need EARL_NVLS=1 at earl_comm_create");
  const uint32_t all = c->world >= 32 ? ~0u : (1u << c->world) - 1u;
  if (team_mask == 0 || (team_mask & ~all) || !(team_mask >> c->rank & 1))
    return fail(EARL_ERR_INVALID_ARGUMENT, "team mask 0x%x: not a subset of the comm containing this rank", team_mask);
  if (c->n_teams >= kMaxShards) return fail(EARL_ERR_CAPACITY, "at most %d multicast teams", kMaxShards);
  if (c->teams[c->n_teams].mc.handle)
    return fail(EARL_ERR_INVALID_ARGUMENT, "a created team must be joined (earl_comm_mc_join) before the next");
  DeviceGuard g(c->device);
  VmmMem mc{0, 0, 0, -1};
  const char* why = "";
  if (!mc_create(__builtin_popcount(team_mask), c->vwin.size, &mc, &why))
    return fail(EARL_ERR_UNSUPPORTED, "cuMulticastCreate(%d devices): %s", __builtin_popcount(team_mask), why);
  FdHandle fh{};
  if (!vmm_export(&mc, &fh.fd, &why)) {
    mc_free(&mc, c->device);
    return fail(EARL_ERR_CUDA, "multicast export: %s", why);
  }
  fh.magic = kTeamMagic;
  fh.pid = (int32_t)getpid();
  fh.size = mc.size;
  fh.mask = team_mask;
  // the creator keeps the object (and its descriptor, until destroy) as a pending team
  c->teams[c->n_teams].mask = 0;  // joined below (earl_comm_mc_join)
  c->teams[c->n_teams].mc = mc;
  std::memset(handle_out, 0, EARL_HANDLE_BYTES);
  std::memcpy(handle_out, &fh, sizeof(fh));
  return EARL_OK;
}

extern "C" earl_status_t earl_comm_mc_join(earl_comm_t c, uint32_t team_mask, const void* handle) {
  if (!c || !handle) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL argument");
  if (!c->vmm) return fail(EARL_ERR_UNSUPPORTED, "multicast teams need EARL_NVLS=1 at earl_comm_create");
  FdHandle fh;
  std::memcpy(&fh, handle, sizeof(fh));
  if (fh.magic != kTeamMagic || fh.mask != team_mask)
    return fail(EARL_ERR_INVALID_ARGUMENT, "not a multicast team handle for mask 0x%x", team_mask);
  if (!(team_mask >> c->rank & 1)) return EARL_OK;  // not a member: nothing to map
  if (c->n_teams >= kMaxShards) return fail(EARL_ERR_CAPACITY, "at most %d multicast teams", kMaxShards);
  DeviceGuard g(c->device);
  earl_comm::Team* t = &c->teams[c->n_teams];
  const char* why = "";
  const bool creator = fh.pid == (int32_t)getpid() && t->mc.handle && t->mask == 0;
  if (!creator) {
    VmmMem mc{0, 0, 0, -1};
    if (!mc_import(fh.pid, fh.fd, fh.size, &mc, &why))
      return fail(EARL_ERR_CUDA, "multicast import: %s", why);
    t->mc = mc;
  }
  if (!mc_join(&t->mc, c->device, c->vwin, &why)) {
    mc_free(&t->mc, c->device);
    return fail(EARL_ERR_UNSUPPORTED, "multicast join: %s", why);
  }
  t->mask = team_mask;
  c->n_teams += 1;
  return EARL_OK;
}

// Plans hold a reference: the comm's resources outlive every plan made on it, whatever order
// the caller (or a garbage collector) destroys them in.
extern "C" earl_status_t earl_comm_destroy(earl_comm_t c) {
  if (!c) return EARL_OK;
  comm_release(c);
  return EARL_OK;
}

// ---------------------------------------------------------------------------------------
// plan
// ---------------------------------------------------------------------------------------

namespace {

earl_status_t check_layout(const earl_layout_t* L, const char* which, int64_t N, int world) {
  if (!L) return fail(EARL_ERR_INVALID_ARGUMENT, "%s layout is NULL", which);
  if (L->dp < 1 || L->sp < 1 || L->tp < 1)
    return fail(EARL_ERR_LAYOUT, "%s layout: dp, sp, tp must be >= 1", which);
  const int64_t nr = (int64_t)L->dp * L->sp * L->tp;
  if (L->rank0 < 0 || L->rank0 + nr > world)
    return fail(EARL_ERR_LAYOUT, "%s layout: ranks [%d, %lld) outside the comm of %d", which,
                L->rank0, (long long)(L->rank0 + nr), world);
  if (L->sp_split < EARL_SP_BLOCK || L->sp_split > EARL_SP_THRESHOLD)
    return fail(EARL_ERR_INVALID_ARGUMENT, "%s layout: unknown sp_split %d", which, L->sp_split);
  if (L->sp_min_len < 0)
    return fail(EARL_ERR_INVALID_ARGUMENT, "%s layout: sp_min_len < 0", which);
  switch (L->assign) {
    case EARL_ASSIGN_GIVEN_COUNTS: {
      if (!L->counts) return fail(EARL_ERR_LAYOUT, "%s layout: GIVEN_COUNTS without counts", which);
      int64_t s = 0;
      for (int g = 0; g < L->dp; ++g) {
        if (L->counts[g] < 0) return fail(EARL_ERR_LAYOUT, "%s layout: negative count", which);
        s += L->counts[g];
      }
      if (s != N)
        return fail(EARL_ERR_LAYOUT, "%s layout: counts sum to %lld, N = %lld", which,
                    (long long)s, (long long)N);
      break;
    }
    case EARL_ASSIGN_CONTIG: break;
    case EARL_ASSIGN_LPT:
      if (N > EARL_LPT_MAX_SEQS)
        return fail(EARL_ERR_CAPACITY, "%s layout: LPT needs N <= %d (N = %lld)", which,
                    EARL_LPT_MAX_SEQS, (long long)N);
      break;
    case EARL_ASSIGN_EXPLICIT:
      if (N > 0 && !L->group_of_seq)
        return fail(EARL_ERR_INVALID_ARGUMENT, "%s layout: EXPLICIT without group_of_seq", which);
      break;
    default: return fail(EARL_ERR_INVALID_ARGUMENT, "%s layout: unknown assign %d", which, L->assign);
  }
  return EARL_OK;
}

LayoutDesc to_desc(const earl_layout_t& L) {
  LayoutDesc d{};
  d.rank0 = L.rank0; d.dp = L.dp; d.sp = L.sp; d.tp = L.tp; d.assign = L.assign;
  d.split = L.sp_split; d.min_len = L.sp_min_len;
  d.group_of_seq = L.group_of_seq;
  d.count_start[0] = 0;
  for (int g = 0; g < L.dp; ++g)
    d.count_start[g + 1] = d.count_start[g] + (L.assign == EARL_ASSIGN_GIVEN_COUNTS ? L.counts[g] : 0);
  return d;
}

template <class T>
T* carve(uint8_t*& p, int64_t count) {
  T* r = reinterpret_cast<T*>(p);
  p += ((size_t)count * sizeof(T) + 255) & ~(size_t)255;
  return r;
}

bool capturing(cudaStream_t s) {
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cap) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return cap != cudaStreamCaptureStatusNone;
}

// Every device launch on a plan is bracketed by use_begin / use_end: a launch on a stream other
// than the plan's last one first waits for the plan's event (the plan's launches share its
// scheduling counters and header, so they are serialised in issue order whatever streams the
// caller uses), and the event is re-recorded after it.  plan_wait and earl_plan_destroy
// therefore cover every launch, not only the planner's.  Under CUDA-graph capture nothing is
// recorded (the caller synchronises the replay stream before host queries, as documented).
void use_begin(earl_plan* p, cudaStream_t s) {
  if (s != p->stream && p->ev && !capturing(s) && p->ev_recorded) cudaStreamWaitEvent(s, p->ev, 0);
}
void use_end(earl_plan* p, cudaStream_t s) {
  p->synced = false;
  if (capturing(s)) return;
  p->stream = s;
  if (p->ev && cudaEventRecord(p->ev, s) == cudaSuccess) p->ev_recorded = true;
}

// Host view of the plan header: always re-read after the plan's last launch completed (a plan
// may have been re-planned on the device -- replan, CUDA-graph replay -- since the last query).
earl_status_t plan_wait(earl_plan_t p) {
  DeviceGuard g(p->comm->device);
  if (p->ev_recorded) CUDA_TRY(cudaEventSynchronize(p->ev));
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  CUDA_TRY(cudaMemcpy(&p->host_hdr, p->args.hdr, sizeof(PlanHeader), cudaMemcpyDeviceToHost));
  p->synced = true;
  return EARL_OK;
}

earl_status_t plan_check(earl_plan_t p) {
  earl_status_t st = plan_wait(p);
  if (st != EARL_OK) return st;
  const PlanHeader& h = p->host_hdr;
  if (h.err != 0) {
    switch (h.err) {
      case EARL_ERR_INVALID_ARGUMENT:
        return fail(EARL_ERR_INVALID_ARGUMENT, "seq_lens[%d] < 0", h.err_detail);
      case EARL_ERR_LAYOUT:
        return fail(EARL_ERR_LAYOUT, "group_of_seq[%d] outside [0, dp)", h.err_detail);
      case EARL_ERR_CAPACITY:
        return fail(EARL_ERR_CAPACITY, "dst shard %d holds more than INT32_MAX tokens", h.err_detail);
      case EARL_ERR_TIMEOUT:
        if ((h.err_detail >> 8) == 0)
          return fail(EARL_ERR_TIMEOUT, "peers missing (mask 0x%x)", h.err_detail & 0xff);
        return fail(EARL_ERR_TIMEOUT,
                    "peers missing (mask 0x%x); peers that skipped their copies (mask 0x%x): this "
                    "rank's receive buffers are incomplete", h.err_detail & 0xff,
                    (h.err_detail >> 8) & 0xff);
      default: return fail((earl_status_t)h.err, "device error %d", h.err_detail);
    }
  }
  return EARL_OK;
}

// (g, k, t) of `rank` in layout L, or false.
bool coords(const earl_layout_t& L, int rank, int* g, int* k, int* t) {
  const int r = rank - L.rank0;
  if (r < 0 || r >= L.dp * L.sp * L.tp) return false;
  *t = r % L.tp;
  *k = (r / L.tp) % L.sp;
  *g = (r / L.tp) / L.sp;
  return true;
}

}  // namespace

// Run the planner into the plan's memory on stream s: reset the header, launch, and record the
// plan's event (not while the stream is being captured into a CUDA graph: the caller then
// synchronises the stream itself before host queries).
cudaError_t plan_launch(earl_plan* p, cudaStream_t s) {
  PlanArgs& a = p->args;
  use_begin(p, s);
  cudaError_t e = cudaMemsetAsync(a.hdr, 0, sizeof(PlanHeader), s);
  if (e != cudaSuccess) return e;
  static const char* plan_trace = getenv("EARL_PLAN_TRACE");
  if (plan_trace) cudaMallocAsync((void**)&a.phase_ts, 16 * sizeof(uint64_t), s);
  clear_stale_error();
  e = launch_planner(a, p->lpt_smem, p->grid, p->fast, s);
  if (plan_trace && e == cudaSuccess) {  // debug only: synchronous read-back of phase times
    uint64_t ts[16];
    cudaMemcpyAsync(ts, a.phase_ts, sizeof(ts), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    if (p->fast) {  // planner_sp1_kernel stamps 0-4 and 7
      fprintf(stderr, "earl plan trace (sp1) N=%lld G=%d us: lengths+reduce %.1f, P+assign %.1f, "
              "histograms %.1f, bases+tables %.1f, emit %.1f, total %.1f\n", (long long)a.N, p->grid,
              (ts[1] - ts[0]) / 1e3, (ts[2] - ts[1]) / 1e3, (ts[3] - ts[2]) / 1e3,
              (ts[4] - ts[3]) / 1e3, (ts[7] - ts[4]) / 1e3, (ts[7] - ts[0]) / 1e3);
      cudaFreeAsync(a.phase_ts, s);
      a.phase_ts = nullptr;
      if (e != cudaSuccess) return e;
      g_launches.fetch_add(1);
      use_end(p, s);
      return cudaSuccess;
    }
    fprintf(stderr, "earl plan trace N=%lld G=%d us:", (long long)a.N, p->grid);
    for (int k = 1; k < 8; ++k) fprintf(stderr, " p%d=%.1f", k - 1, (ts[k] - ts[k - 1]) / 1e3);
    fprintf(stderr, " total=%.1f [p5: loads %.1f, serial %.1f, publish %.1f]", (ts[7] - ts[0]) / 1e3,
            (ts[8] - ts[5]) / 1e3, (ts[9] - ts[8]) / 1e3, (ts[6] - ts[9]) / 1e3);
    fprintf(stderr, " [p2 src: part %.1f, gtok %.1f, scans %.1f; dst: part %.1f, gtok %.1f, scans %.1f]\n",
            (ts[10] - ts[2]) / 1e3, (ts[11] - ts[10]) / 1e3, (ts[12] - ts[11]) / 1e3,
            (ts[13] - ts[12]) / 1e3, (ts[14] - ts[13]) / 1e3, (ts[15] - ts[14]) / 1e3);
    cudaFreeAsync(a.phase_ts, s);
    a.phase_ts = nullptr;
  }
  if (e != cudaSuccess) return e;
  g_launches.fetch_add(1);
  use_end(p, s);
  return cudaSuccess;
}

extern "C" earl_status_t earl_dispatch_plan(earl_comm_t c, const earl_layout_t* src,
                                            const earl_layout_t* dst, const int32_t* seq_lens,
                                            int64_t n_seqs, const earl_field_t* fields,
                                            int32_t n_fields, void* stream, earl_plan_t* out) {
  NvtxRange nvtx("earl_dispatch_plan");
  if (!c || !out) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL comm or plan out-pointer");
  *out = nullptr;
  if (n_seqs < 0 || n_seqs > 0x7fffffffLL)
    return fail(EARL_ERR_INVALID_ARGUMENT, "n_seqs %lld outside [0, 2^31)", (long long)n_seqs);
  if (n_seqs > 0 && !seq_lens) return fail(EARL_ERR_INVALID_ARGUMENT, "seq_lens is NULL");
  if (n_fields < 1 || n_fields > kMaxFields || !fields)
    return fail(EARL_ERR_INVALID_ARGUMENT, "n_fields %d outside [1, %d]", n_fields, kMaxFields);
  for (int f = 0; f < n_fields; ++f) {
    const uint64_t b = (uint64_t)fields[f].bytes_per_elem * fields[f].elems_per_token;
    if (b == 0 || b > (1u << 24))
      return fail(EARL_ERR_INVALID_ARGUMENT, "field %d has %llu bytes per token", f,
                  (unsigned long long)b);
  }
  earl_status_t st;
  if ((st = check_layout(src, "src", n_seqs, c->world)) != EARL_OK) return st;
  if ((st = check_layout(dst, "dst", n_seqs, c->world)) != EARL_OK) return st;
  DeviceGuard g(c->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);

  earl_plan* p = new earl_plan();
  p->comm = c;
  c->refs += 1;
  p->N = n_seqs;
  p->n_fields = n_fields;
  p->stream = s;
  p->lay[0] = *src;
  p->lay[1] = *dst;
  p->lay[0].counts = p->lay[1].counts = nullptr;  // host arrays are consumed now
  std::memcpy(p->fields, fields, sizeof(earl_field_t) * n_fields);

  PlanArgs& a = p->args;
  a.lay[0] = to_desc(*src);
  a.lay[1] = to_desc(*dst);
  a.N = n_seqs;
  a.world = c->world;
  a.n_fields = n_fields;
  for (int f = 0; f < n_fields; ++f) a.Bf[f] = fields[f].bytes_per_elem * fields[f].elems_per_token;
  a.seq_lens = seq_lens;
  const int64_t N = n_seqs;
  const int64_t cs = src->sp_split == EARL_SP_ZIGZAG ? 2 * src->sp : src->sp;
  const int64_t cd = dst->sp_split == EARL_SP_ZIGZAG ? 2 * dst->sp : dst->sp;
  const int64_t max_pieces = N * (cs + cd - 1);
  const int64_t nts = src->tp < dst->tp ? src->tp : dst->tp;
  const int64_t max_records = max_pieces * nts;
  a.max_pieces = max_pieces;
  a.max_records = max_records;

  // size the single allocation (every array 256-B aligned)
  auto sz = [](int64_t count, size_t elem) { return ((size_t)count * elem + 255) & ~(size_t)255; };
  size_t total = sz(1, sizeof(PlanHeader));
  total += sz(N, 4) + sz(N + 1, 8) + 2 * sz(N, 4) + 2 * sz(N, 4);
  total += sz((int64_t)src->sp * N, 8) + sz((int64_t)dst->sp * N, 8);
  total += sz((int64_t)src->sp * (N + 1), 8) + sz((int64_t)dst->sp * (N + 1), 8);
  total += sz(N + 1, 8);
  total += 2 * sz(N, 8) + 2 * sz(N, 4);
  total += 8 * sz(max_pieces, 4) + sz(max_pieces + 1, 8);
  total += sz(kMaxPlanGrid, 8) + sz((int64_t)kMaxPlanGrid * kMaxKeys, 4);
  total += sz((int64_t)2 * kMaxPlanGrid * (kMaxKeys + 2 * kMaxShards), 8);
  const int64_t nscr = (N > max_pieces ? N : max_pieces) + 1;
  total += sz(nscr, 8) + 2 * sz(nscr, 4);
  total += 4 * sz(max_records, 4) + 3 * sz(max_records, 8) + sz(max_records + 1, 8);
  p->mem_bytes = total;
  cudaError_t e = cudaMallocAsync(&p->mem, total, s);
  if (e != cudaSuccess) {
    c->refs -= 1;
    delete p;
    return fail(EARL_ERR_CUDA, "plan cudaMallocAsync(%zu): %s", total, cudaGetErrorString(e));
  }
  uint8_t* q = static_cast<uint8_t*>(p->mem);
  a.hdr = carve<PlanHeader>(q, 1);
  a.lens = carve<int32_t>(q, N);
  a.P = carve<int64_t>(q, N + 1);
  a.grp[0] = carve<int32_t>(q, N);
  a.grp[1] = carve<int32_t>(q, N);
  a.perm[0] = carve<int32_t>(q, N);
  a.perm[1] = carve<int32_t>(q, N);
  a.off[0] = carve<int64_t>(q, (int64_t)src->sp * N);
  a.off[1] = carve<int64_t>(q, (int64_t)dst->sp * N);
  a.cum[0] = carve<int64_t>(q, (int64_t)src->sp * (N + 1));
  a.cum[1] = carve<int64_t>(q, (int64_t)dst->sp * (N + 1));
  a.pbase = carve<int64_t>(q, N + 1);
  a.gpos[0] = carve<int64_t>(q, N);
  a.gpos[1] = carve<int64_t>(q, N);
  a.pos[0] = carve<int32_t>(q, N);
  a.pos[1] = carve<int32_t>(q, N);
  a.pc_i = carve<int32_t>(q, max_pieces);
  a.pc_x = carve<int32_t>(q, max_pieces);
  a.pc_y = carve<int32_t>(q, max_pieces);
  a.pc_kk = carve<int32_t>(q, max_pieces);
  a.ps_i = carve<int32_t>(q, max_pieces);
  a.ps_x = carve<int32_t>(q, max_pieces);
  a.ps_y = carve<int32_t>(q, max_pieces);
  a.ps_kk = carve<int32_t>(q, max_pieces);
  a.ps_scan = carve<int64_t>(q, max_pieces + 1);
  a.cta_sums = carve<int64_t>(q, kMaxPlanGrid);
  a.ghist = carve<int32_t>(q, (int64_t)kMaxPlanGrid * kMaxKeys);
  a.fhist = carve<int64_t>(q, (int64_t)2 * kMaxPlanGrid * (kMaxKeys + 2 * kMaxShards));
  a.vtmp = carve<int64_t>(q, nscr);
  a.ktmp = carve<int32_t>(q, nscr);
  a.ptmp = carve<int32_t>(q, nscr);
  a.rec.seq = carve<int32_t>(q, max_records);
  a.rec.x = carve<int32_t>(q, max_records);
  a.rec.n = carve<int32_t>(q, max_records);
  a.rec.code = carve<uint32_t>(q, max_records);
  a.rec.src_tok = carve<int64_t>(q, max_records);
  a.rec.dst_tok = carve<int64_t>(q, max_records);
  a.rec.msg_tok = carve<int64_t>(q, max_records);
  a.rec.tok_prefix = carve<int64_t>(q, max_records + 1);

  auto abort_plan = [&](earl_status_t code, const char* what, cudaError_t err) {
    cudaFreeAsync(p->mem, s);
    c->refs -= 1;
    delete p;
    return fail(code, "%s: %s", what, cudaGetErrorString(err));
  };
  const bool lpt = src->assign == EARL_ASSIGN_LPT || dst->assign == EARL_ASSIGN_LPT;
  if (lpt) {
    int64_t n2 = 1;
    while (n2 < N) n2 <<= 1;
    p->lpt_smem = (size_t)n2 * sizeof(uint64_t);
  }
  // SP = 1 on both sides (ZIGZAG excepted: its two chunks per sequence are two pieces): the
  // single-pass planner; EARL_PLAN_PATH=general forces the general one (tests compare them)
  const char* path_env = getenv("EARL_PLAN_PATH");
  const bool force_general = path_env && std::strcmp(path_env, "general") == 0;
  p->fast = !force_general && src->sp == 1 && dst->sp == 1 && src->sp_split != EARL_SP_ZIGZAG &&
            dst->sp_split != EARL_SP_ZIGZAG;
  p->grid = planner_grid(N, max_pieces, c->sm_count, p->lpt_smem, p->fast);
  e = cudaEventCreateWithFlags(&p->ev, cudaEventDisableTiming);
  if (e != cudaSuccess) return abort_plan(EARL_ERR_CUDA, "plan event", e);
  e = plan_launch(p, s);
  if (e != cudaSuccess) {
    cudaEventDestroy(p->ev);
    p->ev = nullptr;
    return abort_plan(EARL_ERR_CUDA, "planner launch", e);
  }
  *out = p;
  return EARL_OK;
}

namespace {
// A per-sequence field plan re-reads its token plan's group assignment (stream-ordered after the
// token plan's last launch) before its own planner runs.
cudaError_t refresh_groups(earl_plan* p, cudaStream_t s) {
  earl_plan* t = p->parent;
  const size_t bytes = (size_t)p->N * sizeof(int32_t);
  if (!bytes) return cudaSuccess;
  if (s != t->stream && t->ev_recorded && !capturing(s)) cudaStreamWaitEvent(s, t->ev, 0);
  cudaError_t e = cudaMemcpyAsync(p->owned, t->args.grp[0], bytes, cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(p->owned + p->N, t->args.grp[1], bytes, cudaMemcpyDeviceToDevice, s);
  return e;
}
}  // namespace

extern "C" earl_status_t earl_plan_replan(earl_plan_t p, const int32_t* seq_lens, void* stream) {
  NvtxRange nvtx("earl_plan_replan");
  if (!p) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL plan");
  DeviceGuard g(p->comm->device);
  if (p->parent) {  // a per-sequence field plan: unit lengths, groups from its token plan
    use_begin(p, static_cast<cudaStream_t>(stream));
    cudaError_t e = refresh_groups(p, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return fail(EARL_ERR_CUDA, "replan groups: %s", cudaGetErrorString(e));
    e = plan_launch(p, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return fail(EARL_ERR_CUDA, "replan: %s", cudaGetErrorString(e));
    return EARL_OK;
  }
  if (p->N > 0 && !seq_lens) return fail(EARL_ERR_INVALID_ARGUMENT, "seq_lens is NULL");
  p->args.seq_lens = seq_lens;
  cudaError_t e = plan_launch(p, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(EARL_ERR_CUDA, "replan: %s", cudaGetErrorString(e));
  return EARL_OK;
}

extern "C" earl_status_t earl_plan_sync(earl_plan_t p) {
  if (!p) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL plan");
  p->synced = false;  // re-read: exec may have latched a TIMEOUT
  return plan_check(p);
}

extern "C" earl_status_t earl_plan_local_sizes(earl_plan_t p, int32_t rank, int64_t* n_seqs,
                                               int64_t* n_tokens) {
  if (!p) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL plan");
  earl_status_t st = plan_check(p);
  if (st != EARL_OK) return st;
  int g, k, t;
  int64_t ns = 0, nt = 0;
  if (coords(p->lay[1], rank, &g, &k, &t)) {
    ns = p->host_hdr.group_count[1][g];
    nt = p->host_hdr.shard_tokens[1][g * p->lay[1].sp + k];
  }
  if (n_seqs) *n_seqs = ns;
  if (n_tokens) *n_tokens = nt;
  return EARL_OK;
}

extern "C" earl_status_t earl_plan_local_meta(earl_plan_t p, int32_t rank, int32_t* cu,
                                              int64_t* ids, int32_t* tok_start, void* stream) {
  if (!p) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL plan");
  int g, k, t;
  if (!coords(p->lay[1], rank, &g, &k, &t)) return EARL_OK;  // not a destination: nothing
  DeviceGuard dg(p->comm->device);
  clear_stale_error();
  use_begin(p, (cudaStream_t)stream);
  cudaError_t e = launch_local_meta(p->args, g, k, cu, ids, tok_start, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(EARL_ERR_CUDA, "local_meta launch: %s", cudaGetErrorString(e));
  g_launches.fetch_add(1);
  const bool synced = p->synced;
  use_end(p, (cudaStream_t)stream);
  p->synced = synced;  // a read-only launch: the host header stays valid
  return EARL_OK;
}

extern "C" earl_status_t earl_plan_groups(earl_plan_t p, int32_t* src_groups, int32_t* dst_groups,
                                          void* stream) {
  if (!p) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL plan");
  DeviceGuard dg(p->comm->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t bytes = (size_t)p->N * sizeof(int32_t);
  use_begin(p, s);
  if (bytes && src_groups)
    CUDA_TRY(cudaMemcpyAsync(src_groups, p->args.grp[0], bytes, cudaMemcpyDeviceToDevice, s));
  if (bytes && dst_groups)
    CUDA_TRY(cudaMemcpyAsync(dst_groups, p->args.grp[1], bytes, cudaMemcpyDeviceToDevice, s));
  const bool synced = p->synced;
  use_end(p, s);
  p->synced = synced;
  return EARL_OK;
}

extern "C" earl_status_t earl_plan_mean_length(earl_plan_t p, double* avg) {
  if (!p || !avg) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL argument");
  earl_status_t st = plan_check(p);
  if (st != EARL_OK) return st;
  if (p->N == 0) return fail(EARL_ERR_INVALID_ARGUMENT, "empty batch: no average length");
  *avg = (double)p->host_hdr.T / (double)p->N;
  return EARL_OK;
}

namespace {
// FNV-1a, 64-bit
inline uint64_t fnv1a(uint64_t h, const void* data, size_t n) {
  const unsigned char* b = static_cast<const unsigned char*>(data);
  for (size_t k = 0; k < n; ++k) { h ^= b[k]; h *= 0x100000001b3ull; }
  return h;
}

template <class T>
earl_status_t hash_device(uint64_t& h, const T* dev, int64_t n) {
  if (n <= 0) return EARL_OK;
  std::vector<T> buf((size_t)n);
  CUDA_TRY(cudaMemcpy(buf.data(), dev, sizeof(T) * (size_t)n, cudaMemcpyDeviceToHost));
  h = fnv1a(h, buf.data(), sizeof(T) * (size_t)n);
  return EARL_OK;
}
}  // namespace

extern "C" earl_status_t earl_plan_hash(earl_plan_t p, uint64_t* out) {
  if (!p || !out) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL argument");
  earl_status_t st = plan_check(p);
  if (st != EARL_OK) return st;
  DeviceGuard g(p->comm->device);
  const PlanHeader& h = p->host_hdr;
  uint64_t x = 0xcbf29ce484222325ull;
  // every planned table of the header (not the error latch or the copy kernels' counters)
  const char* lo = reinterpret_cast<const char*>(&h.T);
  const char* hi = reinterpret_cast<const char*>(&h.work_ctr);
  x = fnv1a(x, lo, (size_t)(hi - lo));
  const Records& r = p->args.rec;
  const int64_t n = h.n_records;
  if ((st = hash_device(x, r.seq, n)) != EARL_OK) return st;
  if ((st = hash_device(x, r.x, n)) != EARL_OK) return st;
  if ((st = hash_device(x, r.n, n)) != EARL_OK) return st;
  if ((st = hash_device(x, r.code, n)) != EARL_OK) return st;
  if ((st = hash_device(x, r.src_tok, n)) != EARL_OK) return st;
  if ((st = hash_device(x, r.dst_tok, n)) != EARL_OK) return st;
  if ((st = hash_device(x, r.msg_tok, n)) != EARL_OK) return st;
  if ((st = hash_device(x, r.tok_prefix, n + 1)) != EARL_OK) return st;
  *out = x;
  return EARL_OK;
}

extern "C" earl_status_t earl_plan_stats(earl_plan_t p, earl_plan_stats_t* out) {
  if (!p || !out) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL argument");
  earl_status_t st = plan_check(p);
  if (st != EARL_OK) return st;
  const PlanHeader& h = p->host_hdr;
  const earl_layout_t& S = p->lay[0];
  const earl_layout_t& D = p->lay[1];
  const int W = p->comm->world;
  std::memset(out, 0, sizeof(*out));
  out->world = W;
  out->n_fields = p->n_fields;
  uint64_t B = 0;
  for (int f = 0; f < p->n_fields; ++f) B += p->args.Bf[f];
  out->bytes_per_token = B;
  out->total_tokens = (uint64_t)h.T;
  const int Sd = D.dp * D.sp;
  const int nts = S.tp < D.tp ? S.tp : D.tp;
  int64_t nseg = 0;
  for (int s = 0; s < W; ++s) {
    int gs, ks, ts;
    if (!coords(S, s, &gs, &ks, &ts) || ts >= nts) continue;
    const int ss = gs * S.sp + ks;
    out->stage_bytes[s] = (uint64_t)h.stage_bytes_shard[ss];
    for (int ds = 0; ds < Sd; ++ds) {
      const uint64_t bytes = (uint64_t)h.key_tokens[ss * Sd + ds] * B;
      out->read_bytes[s] += bytes;
      for (int td = ts; td < D.tp; td += S.tp) {
        const int d = D.rank0 + ds * D.tp + td;
        out->C[s][d] += bytes;
        nseg += h.key_pieces[ss * Sd + ds];
      }
    }
  }
  for (int s = 0; s < W; ++s)
    for (int d = 0; d < W; ++d) {
      out->total_bytes += out->C[s][d];
      if (s == d) out->self_bytes[s] += out->C[s][d];
      else { out->egress[s] += out->C[s][d]; out->ingress[d] += out->C[s][d]; }
    }
  for (int r = 0; r < W; ++r) {
    out->moved_bytes += out->egress[r];
    if (out->egress[r] > out->max_egress) out->max_egress = out->egress[r];
    if (out->ingress[r] > out->max_ingress) out->max_ingress = out->ingress[r];
    int g, k, t;
    if (coords(D, r, &g, &k, &t)) {
      out->n_local_seqs[r] = h.group_count[1][g];
      out->n_local_tokens[r] = h.shard_tokens[1][g * D.sp + k];
    }
  }
  out->n_segments = nseg;
  out->n_pieces = h.n_pieces;
  out->n_records = h.n_records;
  return EARL_OK;
}

extern "C" earl_status_t earl_plan_export(earl_plan_t p, int64_t capacity, int64_t* n_segments,
                                          int32_t* s_out, int32_t* d_out, int64_t* seq_out,
                                          int32_t* x_out, int32_t* y_out, int64_t* so_out,
                                          int64_t* do_out) {
  if (!p) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL plan");
  earl_plan_stats_t st;
  earl_status_t r = earl_plan_stats(p, &st);
  if (r != EARL_OK) return r;
  if (n_segments) *n_segments = st.n_segments;
  if (capacity == 0) return EARL_OK;
  if (capacity < st.n_segments)
    return fail(EARL_ERR_CAPACITY, "export capacity %lld < %lld segments", (long long)capacity,
                (long long)st.n_segments);
  if (!s_out || !d_out || !seq_out || !x_out || !y_out || !so_out || !do_out)
    return fail(EARL_ERR_INVALID_ARGUMENT, "export arrays must be non-NULL");
  const PlanHeader& h = p->host_hdr;
  const int64_t M = h.n_records;
  DeviceGuard g(p->comm->device);
  std::vector<int32_t> seq(M), x(M), n(M);
  std::vector<uint32_t> code(M);
  std::vector<int64_t> st_(M), dt(M);
  const Records& R = p->args.rec;
  if (M > 0) {
    CUDA_TRY(cudaMemcpy(seq.data(), R.seq, M * 4, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(x.data(), R.x, M * 4, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(n.data(), R.n, M * 4, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(code.data(), R.code, M * 4, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(st_.data(), R.src_tok, M * 8, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(dt.data(), R.dst_tok, M * 8, cudaMemcpyDeviceToHost));
  }
  // canonical (s, d, i, x): records are (s, ds, i, x); replicas td of a record follow ds.
  const earl_layout_t& S = p->lay[0];
  const earl_layout_t& D = p->lay[1];
  const int Sd = D.dp * D.sp;
  int64_t o = 0;
  for (int s = 0; s < p->comm->world; ++s) {
    int gs, ks, ts;
    if (!coords(S, s, &gs, &ks, &ts)) continue;
    for (int ds = 0; ds < Sd; ++ds) {
      const int64_t b = h.rec_base[s][ds];
      const int64_t e = (ds + 1 < Sd) ? h.rec_base[s][ds + 1] : h.rec_begin[s + 1];
      for (int td = ts; td < D.tp; td += S.tp) {
        const int d = D.rank0 + ds * D.tp + td;
        for (int64_t j = b; j < e; ++j) {
          s_out[o] = s; d_out[o] = d; seq_out[o] = seq[j]; x_out[o] = x[j];
          y_out[o] = x[j] + n[j]; so_out[o] = st_[j]; do_out[o] = dt[j];
          ++o;
        }
      }
    }
  }
  if (o != st.n_segments)
    return fail(EARL_ERR_CUDA, "export produced %lld segments, stats say %lld", (long long)o,
                (long long)st.n_segments);
  return EARL_OK;
}

namespace {
void plan_release(earl_plan* p) {
  if (--p->refs > 0) return;
  {
    DeviceGuard g(p->comm->device);
    if (p->mem) cudaFreeAsync(p->mem, p->stream);
    if (p->owned) cudaFreeAsync(p->owned, p->stream);
    if (p->agg_ws) cudaFree(p->agg_ws);
    if (p->ev) cudaEventDestroy(p->ev);
    cudaGetLastError();
  }
  earl_plan* parent = p->parent;
  comm_release(p->comm);
  delete p;
  if (parent) plan_release(parent);
}
}  // namespace

// A token plan referenced by per-sequence field plans is freed with the last of them.
extern "C" earl_status_t earl_plan_destroy(earl_plan_t p) {
  if (!p) return EARL_OK;
  plan_release(p);
  return EARL_OK;
}

extern "C" earl_status_t earl_plan_seq_fields(earl_plan_t tp, const earl_field_t* fields,
                                              int32_t n_fields, void* stream, earl_plan_t* out) {
  NvtxRange nvtx("earl_plan_seq_fields");
  if (!tp || !out) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL argument");
  *out = nullptr;
  if (tp->parent) return fail(EARL_ERR_INVALID_ARGUMENT, "the plan is itself a per-sequence field plan");
  const int64_t N = tp->N;
  DeviceGuard g(tp->comm->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int32_t* owned = nullptr;
  if (N > 0) {
    CUDA_TRY(cudaMallocAsync(&owned, (size_t)3 * N * sizeof(int32_t), s));
    // unit lengths: one record per sequence
    clear_stale_error();
    cudaError_t e = launch_fill_i32(owned + 2 * N, 1, N, s);
    if (e == cudaSuccess) g_launches.fetch_add(1);
    if (e != cudaSuccess) {
      cudaFreeAsync(owned, s);
      return fail(EARL_ERR_CUDA, "unit lengths: %s", cudaGetErrorString(e));
    }
  }
  // reading n4: the token plan's groups as EXPLICIT layouts, SP folded into TP -- rank (g,k,t) =
  // rank0 + g*sp*tp + k*tp + t is rank (g, 0, k*tp + t) of the folded layout, so every SP rank
  // and TP replica of a group holds one record per sequence of the group
  earl_layout_t fl[2];
  for (int w = 0; w < 2; ++w) {
    fl[w] = tp->lay[w];
    fl[w].tp = tp->lay[w].sp * tp->lay[w].tp;
    fl[w].sp = 1;
    fl[w].assign = EARL_ASSIGN_EXPLICIT;
    fl[w].counts = nullptr;
    fl[w].group_of_seq = owned ? owned + w * N : nullptr;
    fl[w].sp_split = EARL_SP_BLOCK;
    fl[w].sp_min_len = 0;
  }
  earl_plan_t p = nullptr;
  // the planner must see the groups: copy them first (stream-ordered after the token plan)
  earl_plan tmp;
  tmp.parent = tp;
  tmp.N = N;
  tmp.owned = owned;
  use_begin(tp, s);
  cudaError_t e = refresh_groups(&tmp, s);
  tmp.parent = nullptr;
  tmp.owned = nullptr;
  if (e != cudaSuccess) {
    if (owned) cudaFreeAsync(owned, s);
    return fail(EARL_ERR_CUDA, "seq-field groups: %s", cudaGetErrorString(e));
  }
  earl_status_t st = earl_dispatch_plan(tp->comm, &fl[0], &fl[1], owned ? owned + 2 * N : nullptr, N,
                                        fields, n_fields, stream, &p);
  if (st != EARL_OK) {
    if (owned) cudaFreeAsync(owned, s);
    return st;
  }
  p->parent = tp;
  p->owned = owned;
  tp->refs += 1;
  *out = p;
  return EARL_OK;
}

// ---------------------------------------------------------------------------------------
// execution
// ---------------------------------------------------------------------------------------

namespace {

earl_status_t fill_copy_args(earl_plan_t p, CopyArgs& a, int mode) {
  earl_comm* c = p->comm;
  std::memset(&a, 0, sizeof(a));
  const earl_layout_t& S = p->lay[0];
  const earl_layout_t& D = p->lay[1];
  a.mode = mode;
  a.n_fields = p->n_fields;
  a.view_rank = c->emulated ? -1 : c->rank;
  a.nts = S.tp < D.tp ? S.tp : D.tp;
  a.rank0_s = S.rank0; a.tp_s = S.tp;
  a.rank0_d = D.rank0; a.tp_d = D.tp; a.sp_d = D.sp; a.n_dst_shards = D.dp * D.sp;
  a.n_src_shards = S.dp * S.sp;
  a.protocol = 0;
  a.Bpre[0] = 0;
  for (int f = 0; f < p->n_fields; ++f) {
    a.Bf[f] = p->args.Bf[f];
    a.Bpre[f + 1] = a.Bpre[f] + a.Bf[f];
  }
  a.hdr = p->args.hdr;
  a.rec = p->args.rec;
  a.world = c->world;
  a.me = c->emulated ? -1 : c->rank;
  a.peer_mask = node_mask(c);
  a.ds_mask = ~0u;
  a.src_mask = ~0u;
  a.done_ctr = c->done_ctr;
  a.timeout_ns = c->timeout_ns;
  a.err = &p->args.hdr->err;
  a.err_detail = &p->args.hdr->err_detail;
  a.work_ctr = &p->args.hdr->work_ctr;
  a.fin_ctr = &p->args.hdr->fin_ctr;
  return EARL_OK;
}

int copy_grid(earl_comm* c) { return c->sm_count; }

// Debug trace (EARL_COPY_TRACE=<file>): per-warp start/end timestamps of every copy launch,
// appended to <file> as text after a synchronising copy-back.  Never enabled in benchmarks.
struct CopyTrace {
  uint64_t* dev = nullptr;
  size_t n = 0;
  const char* path = nullptr;
};
CopyTrace& trace_state() {
  static CopyTrace t;
  static bool init = false;
  if (!init) { t.path = getenv("EARL_COPY_TRACE"); init = true; }
  return t;
}
// >= 90% of the bytes per token in fields whose width is a multiple of 16 B (always congruent)
int congruent_heavy(const CopyArgs& a) {
  uint64_t cong = 0;
  for (int f = 0; f < a.n_fields; ++f)
    if (a.Bf[f] % 16 == 0) cong += a.Bf[f];
  return cong * 10 >= a.Bpre[a.n_fields] * 9 ? 1 : 0;
}

// The copy-engine shape of a launch: chosen from the field widths (launch_copy), or, for the
// multi-process exec whose stores cross NVLink, forced by EARL_COPY_CFG_P2P (a launch_copy
// shape id; e.g. 3 = 8 warps x 3 x 8 KB, more warps issuing remote stores).
int launch_shape(const CopyArgs& a, const earl_comm* c) {
  static const int p2p_env = [] {
    const char* v = getenv("EARL_COPY_CFG_P2P");
    return v ? atoi(v) : -1;
  }();
  const int p2p = c->opt_p2p_shape >= 0 ? c->opt_p2p_shape : p2p_env;
  if (a.protocol && p2p >= 0) return 100 + p2p;
  return congruent_heavy(a);
}

cudaError_t traced_launch(CopyArgs& a, earl_comm* c, cudaStream_t s) {
  clear_stale_error();
  CopyTrace& t = trace_state();
  if (!t.path) return launch_copy(a, copy_grid(c), launch_shape(a, c), s);
  const size_t n = (size_t)c->sm_count * 64 * 4;
  if (!t.dev) { cudaMalloc(&t.dev, n * 8); t.n = n; }
  cudaMemsetAsync(t.dev, 0, n * 8, s);
  a.trace = t.dev;
  cudaError_t e = launch_copy(a, copy_grid(c), launch_shape(a, c), s);
  if (e != cudaSuccess) return e;
  std::vector<uint64_t> h(n);
  cudaMemcpyAsync(h.data(), t.dev, n * 8, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  FILE* fp = fopen(t.path, "a");
  if (fp) {
    fprintf(fp, "launch mode=%d\n", a.mode);
    for (size_t w = 0; w < n / 4; ++w)
      if (h[4 * w + 1]) fprintf(fp, "%zu %llu %llu %llu %llu\n", w, (unsigned long long)h[4 * w],
                               (unsigned long long)h[4 * w + 1], (unsigned long long)h[4 * w + 2],
                               (unsigned long long)h[4 * w + 3]);
    fclose(fp);
  }
  return cudaSuccess;
}

// Source arrays (direct/pack): emulated [world][F], else [F] for this rank.
earl_status_t set_src(earl_plan_t p, CopyArgs& a, const void* const* bufs) {
  earl_comm* c = p->comm;
  const int F = p->n_fields;
  if (!bufs) return fail(EARL_ERR_INVALID_ARGUMENT, "send_bufs is NULL");
  const int nr = c->emulated ? c->world : 1;
  for (int r = 0; r < nr; ++r) {
    const int rr = c->emulated ? r : c->rank;
    for (int f = 0; f < F; ++f) {
      const void* ptr = bufs[r * F + f];
      if (ptr && !aligned16(ptr))
        return fail(EARL_ERR_INVALID_ARGUMENT, "send buffer rank %d field %d not 16-B aligned", rr, f);
      a.src[rr][f] = static_cast<const uint8_t*>(ptr);
    }
  }
  return EARL_OK;
}

}  // namespace

namespace {

// view: -1 = every record this comm executes (emulated: all source ranks; else this rank's),
// r >= 0 = source rank r's records only (emulated comm)
earl_status_t exec_impl(earl_plan_t p, int view, const void* const* send_bufs,
                        void* const* recv_bufs, void* stream) {
  if (!p) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL plan");
  earl_comm* c = p->comm;
  if (!c->peers_ready)
    return fail(EARL_ERR_INVALID_ARGUMENT, "multi-process comm: earl_comm_import_peers not called");
  if (!recv_bufs) return fail(EARL_ERR_INVALID_ARGUMENT, "recv_bufs is NULL");
  DeviceGuard g(c->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CopyArgs a;
  fill_copy_args(p, a, kDirect);
  if (view >= 0) a.view_rank = view;
  earl_status_t st = set_src(p, a, send_bufs);
  if (st != EARL_OK) return st;
  const int F = p->n_fields;
  if (c->emulated) {
    for (int r = 0; r < c->world; ++r)
      for (int f = 0; f < F; ++f) {
        void* ptr = recv_bufs[r * F + f];
        if (ptr && !aligned16(ptr))
          return fail(EARL_ERR_INVALID_ARGUMENT, "recv buffer rank %d field %d not 16-B aligned", r, f);
        a.dst[r][f] = static_cast<uint8_t*>(ptr);
      }
  } else if (c->world == 1) {
    for (int f = 0; f < F; ++f) {
      void* ptr = recv_bufs[f];
      if (ptr && !aligned16(ptr))
        return fail(EARL_ERR_INVALID_ARGUMENT, "recv buffer field %d not 16-B aligned", f);
      a.dst[0][f] = static_cast<uint8_t*>(ptr);
    }
  } else {
    // every destination publishes its own receive offsets (window-relative) in its signal pad;
    // the entry barrier resolves them into the table the copy kernel stores through, so each
    // rank writes where the DESTINATION put its buffers (NULL = receive nothing)
    uint64_t off[kMaxFields];
    uint8_t* base = c->win[c->rank];
    for (int f = 0; f < F; ++f) {
      uint8_t* ptr = static_cast<uint8_t*>(recv_bufs[f]);
      off[f] = kNoOffset;
      if (!ptr) continue;
      if (!aligned16(ptr))
        return fail(EARL_ERR_INVALID_ARGUMENT, "recv buffer field %d not 16-B aligned", f);
      if (ptr < base + c->pad_bytes || ptr >= base + c->window_bytes)
        return fail(EARL_ERR_INVALID_ARGUMENT,
                    "recv buffer field %d is not inside this rank's window (use earl_comm_alloc)", f);
      off[f] = (uint64_t)(ptr - base);
    }
    a.protocol = 1;
    a.my_pad = reinterpret_cast<uint64_t*>(c->win[c->rank]);
    uint64_t* pads[kMaxWorld] = {};
    for (int q = 0; q < c->world; ++q) pads[q] = reinterpret_cast<uint64_t*>(c->peer[q]);
    for (int q = 0; q < kMaxWorld; ++q) a.peer_pad[q] = pads[q];
    a.dst_tab = reinterpret_cast<uint8_t* const*>(a.my_pad + kDstTabSlot);
    static const int remote_tma = [] {
      const char* v = getenv("EARL_REMOTE_STORE");
      return v && std::strcmp(v, "tma") == 0 ? 1 : 0;
    }();
    a.remote_tma = c->opt_remote_tma >= 0 ? c->opt_remote_tma : remote_tma;
    // NEXT-3: dst shards whose replicas form one of this rank's multicast teams (each source
    // feeds every replica: tp_src == 1); the entry barrier checks the members' offsets agree
    McTeams mct{};
    if (c->n_teams > 0 && a.tp_s == 1 && a.tp_d > 1) {
      for (int ds = 0; ds < a.n_dst_shards && ds < kMaxShards; ++ds) {
        uint32_t want = 0;
        for (int t = 0; t < a.tp_d; ++t) want |= 1u << (a.rank0_d + ds * a.tp_d + t);
        for (int k = 0; k < c->n_teams; ++k)
          if (c->teams[k].mask == want && c->teams[k].mc.va) {
            mct.va[ds] = c->teams[k].mc.va;
            mct.mask[ds] = want;
            a.mc_on = 1;
          }
      }
    }
    a.mc_tab = reinterpret_cast<uint8_t* const*>(a.my_pad + kMcTabSlot);
    use_begin(p, s);
    clear_stale_error();
    cudaError_t e = launch_entry_barrier(a.my_pad, pads, c->world, a.peer_mask, c->rank, F, off,
                                         mct, c->timeout_ns, a.err, a.err_detail, s);
    if (e != cudaSuccess) return fail(EARL_ERR_CUDA, "entry barrier: %s", cudaGetErrorString(e));
    g_launches.fetch_add(1);
  }
  use_begin(p, s);
  cudaError_t e = traced_launch(a, c, s);
  if (e != cudaSuccess) return fail(EARL_ERR_CUDA, "copy launch: %s", cudaGetErrorString(e));
  g_launches.fetch_add(1);
  use_end(p, s);
  return EARL_OK;
}

}  // namespace

extern "C" earl_status_t earl_dispatch_exec(earl_plan_t p, const void* const* send_bufs,
                                            void* const* recv_bufs, void* stream) {
  NvtxRange nvtx("earl_dispatch_exec");
  return exec_impl(p, -1, send_bufs, recv_bufs, stream);
}

extern "C" earl_status_t earl_dispatch_exec_src(earl_plan_t p, int32_t src_rank,
                                                const void* const* send_bufs,
                                                void* const* recv_bufs, void* stream) {
  NvtxRange nvtx("earl_dispatch_exec_src");
  if (!p) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL plan");
  earl_comm* c = p->comm;
  if (src_rank < 0 || src_rank >= c->world)
    return fail(EARL_ERR_INVALID_ARGUMENT, "src_rank %d outside [0, %d)", src_rank, c->world);
  if (!c->emulated) {
    if (src_rank != c->rank)
      return fail(EARL_ERR_INVALID_ARGUMENT, "multi-process comm: src_rank %d is not this rank (%d)",
                  src_rank, c->rank);
    return exec_impl(p, -1, send_bufs, recv_bufs, stream);
  }
  return exec_impl(p, src_rank, send_bufs, recv_bufs, stream);
}

namespace {
// NEXT-4: the destination shards of which this rank feeds a replica on another node
uint32_t remote_shards(earl_plan_t p) {
  const earl_comm* c = p->comm;
  const earl_layout_t& S = p->lay[0];
  const earl_layout_t& D = p->lay[1];
  int g, k, t;
  uint32_t m = 0;
  if (!coords(S, c->rank, &g, &k, &t)) return 0;
  for (int d = 0; d < c->world; ++d) {
    int gd, kd, td;
    if (!coords(D, d, &gd, &kd, &td) || td % S.tp != t) continue;
    if (!same_node(c, d, c->rank)) m |= 1u << (gd * D.sp + kd);
  }
  return m;
}
}  // namespace

extern "C" earl_status_t earl_dispatch_pack(earl_plan_t p, const void* const* send_bufs,
                                            void* const* stage_bufs, void* stream) {
  NvtxRange nvtx("earl_dispatch_pack");
  if (!p || !stage_bufs) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL argument");
  earl_comm* c = p->comm;
  DeviceGuard g(c->device);
  CopyArgs a;
  fill_copy_args(p, a, kPack);
  earl_status_t st = set_src(p, a, send_bufs);
  if (st != EARL_OK) return st;
  const int nr = c->emulated ? c->world : 1;
  for (int r = 0; r < nr; ++r) {
    const int rr = c->emulated ? r : c->rank;
    if (stage_bufs[r] && !aligned16(stage_bufs[r]))
      return fail(EARL_ERR_INVALID_ARGUMENT, "stage buffer %d not 16-B aligned", rr);
    a.stage[rr] = static_cast<uint8_t*>(stage_bufs[r]);
  }
  if (c->node_size > 0) a.ds_mask = remote_shards(p);  // NEXT-4: messages that leave the node
  use_begin(p, static_cast<cudaStream_t>(stream));
  cudaError_t e = traced_launch(a, c, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(EARL_ERR_CUDA, "pack launch: %s", cudaGetErrorString(e));
  g_launches.fetch_add(1);
  use_end(p, static_cast<cudaStream_t>(stream));
  return EARL_OK;
}

extern "C" earl_status_t earl_dispatch_unpack(earl_plan_t p, const void* const* stage_bufs,
                                              void* const* recv_bufs, void* stream) {
  NvtxRange nvtx("earl_dispatch_unpack");
  if (!p || !stage_bufs || !recv_bufs) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL argument");
  earl_comm* c = p->comm;
  DeviceGuard g(c->device);
  CopyArgs a;
  fill_copy_args(p, a, kUnpack);
  const int F = p->n_fields;
  if (c->emulated) {
    for (int r = 0; r < c->world; ++r) {
      if (stage_bufs[r] && !aligned16(stage_bufs[r]))
        return fail(EARL_ERR_INVALID_ARGUMENT, "stage buffer %d not 16-B aligned", r);
      a.stage[r] = const_cast<uint8_t*>(static_cast<const uint8_t*>(stage_bufs[r]));
      for (int f = 0; f < F; ++f) {
        void* ptr = recv_bufs[r * F + f];
        if (ptr && !aligned16(ptr))
          return fail(EARL_ERR_INVALID_ARGUMENT, "recv buffer rank %d field %d not 16-B aligned", r, f);
        a.dst[r][f] = static_cast<uint8_t*>(ptr);
      }
    }
  } else {
    // a real rank: stage_bufs[0] holds the messages it received, concatenated in source-rank
    // order (earl_plan_messages gives each one's offset); recv_bufs[F] are its field arrays
    if (stage_bufs[0] && !aligned16(stage_bufs[0]))
      return fail(EARL_ERR_INVALID_ARGUMENT, "receive stage buffer not 16-B aligned");
    a.recv_stage = static_cast<const uint8_t*>(stage_bufs[0]);
    for (int f = 0; f < F; ++f) {
      void* ptr = recv_bufs[f];
      if (ptr && !aligned16(ptr))
        return fail(EARL_ERR_INVALID_ARGUMENT, "recv buffer field %d not 16-B aligned", f);
      a.dst[c->rank][f] = static_cast<uint8_t*>(ptr);
    }
    if (c->node_size > 0) a.src_mask = ~node_mask(c);  // NEXT-4: messages from other nodes
  }
  use_begin(p, static_cast<cudaStream_t>(stream));
  cudaError_t e = traced_launch(a, c, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(EARL_ERR_CUDA, "unpack launch: %s", cudaGetErrorString(e));
  g_launches.fetch_add(1);
  use_end(p, static_cast<cudaStream_t>(stream));
  return EARL_OK;
}

namespace {
// The staged path's per-peer byte table of `rank` from the plan's (synced) host header.
void message_table(earl_plan_t p, int rank, int64_t* send_off, int64_t* send_bytes,
                   int64_t* recv_off, int64_t* recv_bytes) {
  const int W = p->comm->world;
  const PlanHeader& h = p->host_hdr;
  const earl_layout_t& S = p->lay[0];
  const earl_layout_t& D = p->lay[1];
  const int Sd = D.dp * D.sp;
  const int nts = S.tp < D.tp ? S.tp : D.tp;
  auto msg_bytes = [&](int key) {
    int64_t b = 0;
    for (int f = 0; f < p->n_fields; ++f) b += ((int64_t)h.key_tokens[key] * p->args.Bf[f] + 15) & ~15LL;
    return b;
  };
  for (int q = 0; q < W; ++q) { send_off[q] = send_bytes[q] = recv_off[q] = recv_bytes[q] = 0; }
  const earl_comm* c = p->comm;
  int g, k, t;
  // sends: this rank's message to dst shard ds goes to every replica td == ts (mod tp_src);
  // a multi-node comm (NEXT-4) stages only the messages that leave the node
  if (coords(S, rank, &g, &k, &t) && t < nts) {
    const int ss = g * S.sp + k;
    for (int d = 0; d < W; ++d) {
      int gd, kd, td;
      if (!coords(D, d, &gd, &kd, &td) || td % S.tp != t) continue;
      if (c->node_size > 0 && same_node(c, d, rank)) continue;
      const int ds = gd * D.sp + kd;
      send_off[d] = h.msg_off[ss * Sd + ds];
      send_bytes[d] = msg_bytes(ss * Sd + ds);
    }
  }
  // receives: concatenated in source-rank order
  if (coords(D, rank, &g, &k, &t)) {
    const int ds = g * D.sp + k;
    int64_t off = 0;
    for (int s = 0; s < W; ++s) {
      int gs, ks, ts;
      if (!coords(S, s, &gs, &ks, &ts) || ts >= nts || t % S.tp != ts) continue;
      if (c->node_size > 0 && same_node(c, s, rank)) continue;
      const int key = (gs * S.sp + ks) * Sd + ds;
      recv_off[s] = off;
      recv_bytes[s] = msg_bytes(key);
      off += recv_bytes[s];
    }
  }
}
}  // namespace

extern "C" earl_status_t earl_plan_messages(earl_plan_t p, int32_t rank, int64_t* send_off,
                                            int64_t* send_bytes, int64_t* recv_off,
                                            int64_t* recv_bytes) {
  if (!p || !send_off || !send_bytes || !recv_off || !recv_bytes)
    return fail(EARL_ERR_INVALID_ARGUMENT, "NULL argument");
  const int W = p->comm->world;
  if (rank < 0 || rank >= W) return fail(EARL_ERR_INVALID_ARGUMENT, "rank %d outside the comm", rank);
  earl_status_t st = plan_check(p);
  if (st != EARL_OK) return st;
  message_table(p, rank, send_off, send_bytes, recv_off, recv_bytes);
  return EARL_OK;
}

// ---------------------------------------------------------------------------------------
// K8: the staged exchange over NCCL (grouped ncclSend / ncclRecv), the comparator of the fused
// P2P exec
// ---------------------------------------------------------------------------------------

#define NCCL_TRY(expr)                                                                     \
  do {                                                                                     \
    ncclResult_t r_ = (expr);                                                              \
    if (r_ != ncclSuccess)                                                                 \
      return fail(EARL_ERR_NCCL, "%s failed: %s (%s)", #expr, ncclGetErrorString(r_),      \
                  ncclGetLastError(nullptr));                                              \
  } while (0)

extern "C" earl_status_t earl_nccl_unique_id(void* id_out) {
  if (!id_out) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL argument");
  static_assert(sizeof(ncclUniqueId) <= EARL_HANDLE_BYTES, "unique id size");
  ncclUniqueId id;
  NCCL_TRY(ncclGetUniqueId(&id));
  std::memset(id_out, 0, EARL_HANDLE_BYTES);
  std::memcpy(id_out, &id, sizeof(id));
  return EARL_OK;
}

extern "C" earl_status_t earl_comm_init_nccl(earl_comm_t c, const void* unique_id) {
  if (!c || !unique_id) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL argument");
  if (c->emulated) return fail(EARL_ERR_UNSUPPORTED, "emulated comm: the NCCL exchange needs one process per GPU");
  if (c->nccl) return EARL_OK;
  DeviceGuard g(c->device);
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
  if (const char* v = getenv("EARL_NCCL_MIN_CTAS")) cfg.minCTAs = atoi(v);
  if (const char* v = getenv("EARL_NCCL_MAX_CTAS")) cfg.maxCTAs = atoi(v);
  cfg.commName = "earl_dispatch";
  NCCL_TRY(ncclCommInitRankConfig(&c->nccl, c->world, id, c->rank, &cfg));
  const char* reg = getenv("EARL_NCCL_REGISTER");
  c->nccl_register = reg && atoi(reg) != 0;
  return EARL_OK;
}

namespace {
// Grow stage buffer k (0 = send, 1 = receive) of the comm to at least `bytes`.
earl_status_t nccl_stage(earl_comm* c, int k, uint64_t bytes) {
  if (bytes < 16) bytes = 16;
  if (c->nst[k] && c->nst_bytes[k] >= bytes) return EARL_OK;
  CUDA_TRY(cudaDeviceSynchronize());  // the old buffer may still be in use
  if (c->nreg[k]) { ncclCommDeregister(c->nccl, c->nreg[k]); c->nreg[k] = nullptr; }
  if (c->nst[k]) {
    if (c->nccl_register) ncclMemFree(c->nst[k]);
    else cudaFree(c->nst[k]);
    c->nst[k] = nullptr;
  }
  bytes = (bytes + (1ull << 21) - 1) & ~((1ull << 21) - 1);
  if (c->nccl_register) {
    NCCL_TRY(ncclMemAlloc(&c->nst[k], bytes));
    NCCL_TRY(ncclCommRegister(c->nccl, c->nst[k], bytes, &c->nreg[k]));
  } else {
    CUDA_TRY(cudaMalloc(&c->nst[k], bytes));
  }
  c->nst_bytes[k] = bytes;
  return EARL_OK;
}
}  // namespace

namespace {
// The grouped send/recv of this rank's messages (the plan's host header must be current).
earl_status_t exchange_impl(earl_plan_t p, const void* send_stage, void* recv_stage, void* stream) {
  earl_comm* c = p->comm;
  const int W = c->world;
  int64_t so[kMaxWorld], sb[kMaxWorld], ro[kMaxWorld], rb[kMaxWorld];
  message_table(p, c->rank, so, sb, ro, rb);
  int64_t need_s = 0, need_r = 0;
  for (int q = 0; q < W; ++q) {
    if (sb[q]) need_s = std::max(need_s, so[q] + sb[q]);
    if (rb[q]) need_r = std::max(need_r, ro[q] + rb[q]);
  }
  if ((need_s && !send_stage) || (need_r && !recv_stage))
    return fail(EARL_ERR_INVALID_ARGUMENT, "stage buffer is NULL");
  DeviceGuard g(c->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint8_t* sp = static_cast<const uint8_t*>(send_stage);
  uint8_t* rp = static_cast<uint8_t*>(recv_stage);
  use_begin(p, s);
  NCCL_TRY(ncclGroupStart());
  for (int q = 0; q < W; ++q) {
    if (sb[q]) NCCL_TRY(ncclSend(sp + so[q], (size_t)sb[q], ncclUint8, q, c->nccl, s));
    if (rb[q]) NCCL_TRY(ncclRecv(rp + ro[q], (size_t)rb[q], ncclUint8, q, c->nccl, s));
  }
  NCCL_TRY(ncclGroupEnd());
  use_end(p, s);
  return EARL_OK;
}
}  // namespace

extern "C" earl_status_t earl_dispatch_exchange(earl_plan_t p, const void* send_stage,
                                                void* recv_stage, void* stream) {
  NvtxRange nvtx("earl_dispatch_exchange");
  if (!p) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL plan");
  if (!p->comm->nccl) return fail(EARL_ERR_INVALID_ARGUMENT, "earl_comm_init_nccl was not called");
  earl_status_t st = plan_check(p);  // the byte table is host data: NCCL takes host sizes
  if (st != EARL_OK) return st;
  return exchange_impl(p, send_stage, recv_stage, stream);
}

extern "C" earl_status_t earl_dispatch_exec_staged(earl_plan_t p, const void* const* send_bufs,
                                                   void* const* recv_bufs, void* stream) {
  NvtxRange nvtx("earl_dispatch_exec_staged");
  if (!p) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL plan");
  earl_comm* c = p->comm;
  if (!c->nccl) return fail(EARL_ERR_INVALID_ARGUMENT, "earl_comm_init_nccl was not called");
  earl_status_t st = plan_check(p);
  if (st != EARL_OK) return st;
  int64_t so[kMaxWorld], sb[kMaxWorld], ro[kMaxWorld], rb[kMaxWorld];
  message_table(p, c->rank, so, sb, ro, rb);
  int64_t need_r = 0;
  for (int q = 0; q < c->world; ++q) need_r += rb[q];
  int gs, ks, ts;
  const int64_t need_s = coords(p->lay[0], c->rank, &gs, &ks, &ts) ? p->host_hdr.stage_bytes_shard[gs * p->lay[0].sp + ks] : 0;
  DeviceGuard g(c->device);
  if ((st = nccl_stage(c, 0, (uint64_t)need_s)) != EARL_OK) return st;
  if ((st = nccl_stage(c, 1, (uint64_t)need_r)) != EARL_OK) return st;
  void* stage_s[1] = {c->nst[0]};
  void* stage_r[1] = {c->nst[1]};
  if ((st = earl_dispatch_pack(p, send_bufs, stage_s, stream)) != EARL_OK) return st;
  if ((st = exchange_impl(p, c->nst[0], c->nst[1], stream)) != EARL_OK) return st;
  return earl_dispatch_unpack(p, stage_r, recv_bufs, stream);
}

extern "C" earl_status_t earl_dispatch_exec_hier(earl_plan_t p, const void* const* send_bufs,
                                                 void* const* recv_bufs, void* stream) {
  NvtxRange nvtx("earl_dispatch_exec_hier");
  if (!p) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL plan");
  if (p->comm->node_size == 0)
    return fail(EARL_ERR_INVALID_ARGUMENT, "earl_comm_set_nodes was not called (one node: use earl_dispatch_exec)");
  earl_status_t st = exec_impl(p, -1, send_bufs, recv_bufs, stream);  // inside the node: fused P2P
  if (st != EARL_OK) return st;
  return earl_dispatch_exec_staged(p, send_bufs, recv_bufs, stream);  // across nodes: NCCL
}

// ---------------------------------------------------------------------------------------
// NEXT-2: distributed advantage estimation on the source ranks (aggregate.cu)
// ---------------------------------------------------------------------------------------

namespace {

earl_status_t agg_args(earl_plan_t p, AggArgs& a) {
  std::memset(&a, 0, sizeof(a));
  if (p->lay[0].sp != 1)
    return fail(EARL_ERR_UNSUPPORTED, "returns/advantages need whole sequences on the source (sp == 1)");
  a.plan = p->args;
  a.hdr = p->args.hdr;
  a.world = p->comm->world;
  a.view_rank = p->comm->emulated ? -1 : p->comm->rank;
  return EARL_OK;
}

// The look-back workspace of returns_kernel: allocated (zeroed) on first use, outside any graph
// capture, for at least 2^20 windows (2^30 tokens per source rank set) or the plan's known token
// count; the kernel latches EARL_ERR_CAPACITY in the plan header beyond it.
earl_status_t agg_workspace(earl_plan_t p, cudaStream_t s) {
  int64_t need = int64_t(1) << 20;
  if (p->synced) need = std::max(need, returns_windows(p->host_hdr.T) + kMaxWorld);
  if (p->agg_ws && p->agg_cap >= need) return EARL_OK;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CUDA_TRY(cudaStreamIsCapturing(s, &cs));
  if (cs != cudaStreamCaptureStatusNone)
    return fail(EARL_ERR_UNSUPPORTED,
                "the first earl_returns on a plan allocates its workspace: call it once before graph capture");
  if (p->agg_ws) {
    CUDA_TRY(cudaFree(p->agg_ws));
    p->agg_ws = nullptr;
  }
  // AggWork | AggWindow[need] (windowed kernel) | int64 unit_first[need] (unit kernel)
  const size_t bytes = sizeof(AggWork) + (sizeof(AggWindow) + sizeof(int64_t)) * (size_t)need;
  CUDA_TRY(cudaMalloc(&p->agg_ws, bytes));
  p->agg_cap = need;
  CUDA_TRY(cudaMemsetAsync(p->agg_ws, 0, bytes, s));
  return EARL_OK;
}

template <class T>
earl_status_t set_per_rank(earl_plan_t p, T** dst, const void* const* src, const char* what,
                           bool required) {
  earl_comm* c = p->comm;
  if (!src) {
    if (required) return fail(EARL_ERR_INVALID_ARGUMENT, "%s is NULL", what);
    return EARL_OK;
  }
  const int nr = c->emulated ? c->world : 1;
  for (int r = 0; r < nr; ++r) {
    const int rr = c->emulated ? r : c->rank;
    dst[rr] = const_cast<T*>(static_cast<const T*>(src[r]));
  }
  return EARL_OK;
}

}  // namespace

extern "C" earl_status_t earl_returns(earl_plan_t p, float gamma, const void* const* rewards,
                                      const void* const* mask, void* const* returns,
                                      void* const* seq_return, double* partial, void* stream) {
  NvtxRange nvtx("earl_returns");
  if (!p || !partial) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL argument");
  AggArgs a;
  earl_status_t st = agg_args(p, a);
  if (st != EARL_OK) return st;
  a.gamma = gamma;
  a.gamma16 = 1.f;
  for (int i = 0; i < 16; ++i) a.gamma16 *= gamma;
  a.gpw[0] = a.gamma16;
  for (int k = 1; k < 5; ++k) a.gpw[k] = a.gpw[k - 1] * a.gpw[k - 1];
  a.g4 = (gamma * gamma) * (gamma * gamma);
  a.g512 = a.gpw[4] * a.gpw[4];
  a.partial = partial;
  if ((st = set_per_rank<const float>(p, a.rewards, rewards, "rewards", true)) != EARL_OK) return st;
  if ((st = set_per_rank<const uint8_t>(p, a.mask, mask, "mask", true)) != EARL_OK) return st;
  if ((st = set_per_rank<float>(p, a.returns, (const void* const*)returns, "returns", true)) != EARL_OK) return st;
  if ((st = set_per_rank<float>(p, a.seq_return, (const void* const*)seq_return, "seq_return", false)) != EARL_OK)
    return st;
  DeviceGuard g(p->comm->device);
  clear_stale_error();
  if ((st = agg_workspace(p, static_cast<cudaStream_t>(stream))) != EARL_OK) return st;
  a.ws = static_cast<AggWork*>(p->agg_ws);
  a.win = reinterpret_cast<AggWindow*>(a.ws + 1);
  a.win_cap = p->agg_cap;
  a.unit_first = reinterpret_cast<int64_t*>(a.win + p->agg_cap);
  // Three returns kernels (choose_returns): the cooperative one when every window of the batch
  // gets its own warp of a co-resident grid (small and mid batches), the single-pass unit kernel
  // for large batches without sequences longer than kUnitMaxLen, else the windowed look-back
  // kernel.  The host decides when it knows the batch; otherwise every kernel is launched and
  // each evaluates the rule on the device from the plan header (all but one exit at once).
  // EARL_RETURNS=coop|units|windows forces one (tests).
  const char* force = getenv("EARL_RETURNS");
  a.resident_warps = (int64_t)p->comm->sm_count * kUnitWarpsPerSm;
  a.coop_warps = returns_coop_capacity_warps(p->comm->sm_count);
  a.coop_nb = 0;
  int kmask = a.coop_warps > 0 ? 7 : 3;  // bit k: launch kernel k (ReturnsKernel)
  int64_t coop_need = 0;                // the cooperative kernel's windows (0: its whole grid)
  if (p->synced) {
    const earl_layout_t& S = p->lay[0];
    int64_t nt[kMaxWorld];
    int n = 0;
    for (int r = 0; r < p->comm->world; ++r) {
      if (!p->comm->emulated && r != p->comm->rank) continue;
      const int q = r - S.rank0;
      if (q < 0 || q >= S.dp * S.tp) continue;
      nt[n++] = p->host_hdr.shard_tokens[0][q / S.tp];
    }
    int nb = 0;
    const int id = choose_returns(nt, n, p->host_hdr.max_len, a.resident_warps, a.coop_warps, &nb);
    kmask = 1 << id;
    if (nb > 0) {
      a.coop_nb = nb;
      for (int i = 0; i < n; ++i) coop_need += (nt[i] + 512LL * nb - 1) / (512LL * nb);
    }
  }
  if (force && std::strcmp(force, "units") == 0) kmask = 1 << kRetUnits;
  if (force && std::strcmp(force, "windows") == 0) kmask = 1 << kRetWindows;
  if (force && std::strcmp(force, "coop") == 0) kmask = 1 << kRetCoop;
  const bool gated = (kmask & (kmask - 1)) != 0;
  cudaStream_t rs = static_cast<cudaStream_t>(stream);
  use_begin(p, rs);
  cudaError_t e = cudaSuccess;
  if (kmask & (1 << kRetCoop)) {
    a.gate = gated ? kRetCoop + 1 : 0;
    e = launch_returns_coop(a, coop_need, p->comm->sm_count, rs);
    if (e == cudaSuccess) g_launches.fetch_add(1);
  }
  if (e == cudaSuccess && (kmask & (1 << kRetUnits))) {
    a.gate = gated ? kRetUnits + 1 : 0;
    e = launch_returns_units(a, p->comm->sm_count, rs);
    if (e == cudaSuccess) g_launches.fetch_add(2);  // the unit table kernel, the unit kernel
  }
  if (e == cudaSuccess && (kmask & (1 << kRetWindows))) {
    a.gate = gated ? kRetWindows + 1 : 0;
    e = launch_returns(a, p->comm->sm_count, rs);
    if (e == cudaSuccess) g_launches.fetch_add(1);
  }
  if (e != cudaSuccess) return fail(EARL_ERR_CUDA, "returns launch: %s", cudaGetErrorString(e));
  const bool synced = p->synced;
  use_end(p, static_cast<cudaStream_t>(stream));
  p->synced = synced;  // T is unchanged (a CAPACITY latch is read by the next synchronising call)
  return EARL_OK;
}

extern "C" earl_status_t earl_advantages(earl_plan_t p, const double* stats, float eps,
                                         const void* const* returns, const void* const* mask,
                                         void* const* adv, void* stream) {
  NvtxRange nvtx("earl_advantages");
  if (!p || !stats) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL argument");
  AggArgs a;
  earl_status_t st = agg_args(p, a);
  if (st != EARL_OK) return st;
  a.stats = stats;
  a.eps = eps;
  if ((st = set_per_rank<float>(p, a.returns, returns, "returns", true)) != EARL_OK) return st;
  if ((st = set_per_rank<const uint8_t>(p, a.mask, mask, "mask", true)) != EARL_OK) return st;
  if ((st = set_per_rank<float>(p, a.adv, (const void* const*)adv, "adv", true)) != EARL_OK) return st;
  DeviceGuard g(p->comm->device);
  clear_stale_error();
  // the source ranks' tokens this launch covers, when the host knows the plan (else -1)
  int64_t tokens = -1;
  if (p->synced) {
    const earl_layout_t& S = p->lay[0];
    tokens = p->comm->emulated ? p->host_hdr.T * S.tp : (p->host_hdr.T + S.dp - 1) / S.dp;
  }
  use_begin(p, static_cast<cudaStream_t>(stream));
  cudaError_t e = launch_advantages(a, p->comm->sm_count, tokens, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(EARL_ERR_CUDA, "advantages launch: %s", cudaGetErrorString(e));
  g_launches.fetch_add(1);
  const bool synced = p->synced;
  use_end(p, static_cast<cudaStream_t>(stream));
  p->synced = synced;
  return EARL_OK;
}
