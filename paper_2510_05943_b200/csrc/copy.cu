// copy.cu -- the byte-moving kernels of the dispatcher (SURVEY.md §8(a) a3 pack, a5 unpack,
// a6 fused direct/P2P, a7 completion).
//
// All three modes run the same persistent kernel over the plan's copy records.  The work of a
// launch is the field-major byte space  sum_f Ntok * B_f  (Ntok = tokens of the records in
// the launch's view); every warp takes one contiguous, equal slice of it, so a 32K-token
// sequence next to hundreds of 100-token ones is split by bytes, not by sequence.  A warp
// finds its first record by binary search over the records' token prefix and then walks
// records in order.  Each (record, field) piece is copied by warp_copy: 16-B vector stores on
// the destination, 16-B vector loads on the source realigned in registers (warp shuffle +
// funnel shift) when source and destination differ mod 16 -- the 4-B id/fp32 fields and 1-B
// masks start at arbitrary token offsets.  Replicated destinations (TP, reading c2) are
// written from the same registers: each source byte is read once.  No tensor cores: the path
// is pure data movement (HBM roofline).
#include "earl_internal.cuh"

namespace earl {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kUnroll = 4;

__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_v4(void* p, const uint4& v) {
  *reinterpret_cast<uint4*>(p) = v;
}

__device__ __forceinline__ uint4 shfl_down4(const uint4& v, int d) {
  return make_uint4(__shfl_down_sync(kFull, v.x, d), __shfl_down_sync(kFull, v.y, d),
                    __shfl_down_sync(kFull, v.z, d), __shfl_down_sync(kFull, v.w, d));
}
__device__ __forceinline__ uint4 shfl_idx4(const uint4& v, int src) {
  return make_uint4(__shfl_sync(kFull, v.x, src), __shfl_sync(kFull, v.y, src),
                    __shfl_sync(kFull, v.z, src), __shfl_sync(kFull, v.w, src));
}

// 16 bytes starting at byte sh (1..15) of the 32-byte pair (A, B).  s4 = sh/4 and
// bits = 8*(sh%4) are warp-uniform (they depend on the source address only).
__device__ __forceinline__ uint4 realign(const uint4& A, const uint4& B, int s4, int bits) {
  uint32_t v0, v1, v2, v3, v4;
  switch (s4) {
    case 0: v0 = A.x; v1 = A.y; v2 = A.z; v3 = A.w; v4 = B.x; break;
    case 1: v0 = A.y; v1 = A.z; v2 = A.w; v3 = B.x; v4 = B.y; break;
    case 2: v0 = A.z; v1 = A.w; v2 = B.x; v3 = B.y; v4 = B.z; break;
    default: v0 = A.w; v1 = B.x; v2 = B.y; v3 = B.z; v4 = B.w; break;
  }
  return make_uint4(__funnelshift_r(v0, v1, bits), __funnelshift_r(v1, v2, bits),
                    __funnelshift_r(v2, v3, bits), __funnelshift_r(v3, v4, bits));
}

// Copy len bytes from src to each of dst[0..R) (all destinations share the same alignment
// mod 16 -- field bases are 16-B aligned and replicas use the same token offset).
// Called by a whole warp with warp-uniform arguments.
__device__ __forceinline__ void warp_copy(const uint8_t* __restrict__ src, uint8_t* const* dst,
                                          int R, int64_t len, int lane) {
  if (len <= 0) return;
  int64_t head = (16 - ((uintptr_t)dst[0] & 15)) & 15;
  if (head > len) head = len;
  if (lane < head) {
    const uint8_t v = src[lane];
    for (int r = 0; r < R; ++r) dst[r][lane] = v;
  }
  const uint8_t* s = src + head;
  const int64_t dofs = head;
  const int64_t rest = len - head;
  const int64_t nvec = rest >> 4;
  if (nvec > 0) {
    const int sh = (int)((uintptr_t)s & 15);
    if (sh == 0) {
      const uint4* sp = reinterpret_cast<const uint4*>(s);
      for (int64_t base = 0; base < nvec; base += 32 * kUnroll) {
        uint4 v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const int64_t c = base + u * 32 + lane;
          if (c < nvec) v[u] = ld_stream(sp + c);
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const int64_t c = base + u * 32 + lane;
          if (c < nvec)
            for (int r = 0; r < R; ++r) st_v4(dst[r] + dofs + c * 16, v[u]);
        }
      }
    } else {
      // Source words sal[c] and sal[c+1] hold destination chunk c.  Word nvec contains valid
      // source bytes whenever sh > 0, so loading it never leaves the source allocation.
      const uint4* sal = reinterpret_cast<const uint4*>(s - sh);
      const int s4 = sh >> 2, bits = (sh & 3) * 8;
      for (int64_t base = 0; base < nvec; base += 32 * kUnroll) {
        uint4 A[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const int64_t c = base + u * 32 + lane;
          A[u] = (c <= nvec) ? ld_stream(sal + c) : make_uint4(0, 0, 0, 0);
        }
        uint4 extra = make_uint4(0, 0, 0, 0);
        const int64_t ce = base + 32 * kUnroll;
        if (lane == 31 && ce <= nvec) extra = ld_stream(sal + ce);
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const uint4 dn = shfl_down4(A[u], 1);
          const uint4 nx = (u + 1 < kUnroll) ? shfl_idx4(A[(u + 1) % kUnroll], 0) : extra;
          const uint4 B = (lane == 31) ? nx : dn;
          const int64_t c = base + u * 32 + lane;
          if (c < nvec) {
            const uint4 o = realign(A[u], B, s4, bits);
            for (int r = 0; r < R; ++r) st_v4(dst[r] + dofs + c * 16, o);
          }
        }
      }
    }
  }
  const int64_t done = nvec << 4;
  const int64_t tail = rest - done;
  if (lane < tail) {
    const uint8_t v = s[done + lane];
    for (int r = 0; r < R; ++r) dst[r][dofs + done + lane] = v;
  }
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Signal every peer (slot `slot_base + me` of its pad), then wait for every peer's signal in
// my pad.  Lane p handles peer p.  Returns the mask of peers that timed out.
__device__ unsigned signal_and_wait(uint64_t* my_pad, uint64_t* const* peer_pad, int world, int me,
                                    int slot_base, uint64_t epoch, uint64_t timeout_ns) {
  const int lane = threadIdx.x & 31;
  if (lane < world && lane != me) st_release_sys(peer_pad[lane] + slot_base + me, epoch);
  unsigned missing = 0;
  if (lane < world && lane != me) {
    const uint64_t t0 = globaltimer();
    while (ld_acquire_sys(my_pad + slot_base + lane) < epoch) {
      if (globaltimer() - t0 > timeout_ns) { missing = 1u << lane; break; }
      __nanosleep(64);
    }
  }
  return __reduce_or_sync(kFull, missing);
}

__global__ void entry_barrier_kernel(uint64_t* my_pad, PeerPads pads, int world, int me,
                                     uint64_t epoch, uint64_t timeout_ns, int32_t* err,
                                     int32_t* err_detail) {
  const unsigned miss = signal_and_wait(my_pad, pads.p, world, me, kReadySlot, epoch, timeout_ns);
  if (threadIdx.x == 0 && miss) {
    if (atomicCAS(err, 0, EARL_ERR_TIMEOUT) == 0) *err_detail = (int32_t)miss;
  }
}

__global__ void __launch_bounds__(512, 2) copy_kernel(const CopyArgs a) {
  __shared__ unsigned s_last;
  const PlanHeader* h = a.hdr;
  const int lane = threadIdx.x & 31;
  const int F = a.n_fields;
  if (h->err == 0) {
    int64_t rbeg, rend, tbeg, tend;
    if (a.view_rank < 0) {
      rbeg = 0; rend = h->n_records; tbeg = 0; tend = h->rec_tokens;
    } else {
      rbeg = h->rec_begin[a.view_rank]; rend = h->rec_begin[a.view_rank + 1];
      tbeg = h->rec_tok_begin[a.view_rank]; tend = h->rec_tok_begin[a.view_rank + 1];
    }
    const uint64_t ntok = (uint64_t)(tend - tbeg);
    const uint64_t total = ntok * a.Bpre[F];
    const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    const uint64_t wid = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const uint64_t chunk = (((total + nwarps - 1) / nwarps) + 511) & ~511ull;
    const uint64_t b0 = wid * chunk;
    const uint64_t b1 = (b0 + chunk < total) ? b0 + chunk : total;
    if (b0 < b1) {
      int f = 0;
      while (b0 >= ntok * a.Bpre[f + 1]) ++f;
      const int64_t tok = tbeg + (int64_t)((b0 - ntok * a.Bpre[f]) / a.Bf[f]);
      // last record j in [rbeg, rend) with tok_prefix[j] <= tok
      int64_t lo = rbeg, hi = rend - 1;
      while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (a.rec.tok_prefix[mid] <= tok) lo = mid; else hi = mid - 1;
      }
      int64_t j = lo;
      uint64_t pos = b0;
      const int Sd = a.n_dst_shards;
      while (pos < b1) {
        const uint64_t Bf = a.Bf[f];
        const uint64_t fs = ntok * a.Bpre[f];
        const int64_t tp0 = a.rec.tok_prefix[j] - tbeg;
        const int64_t tp1 = a.rec.tok_prefix[j + 1] - tbeg;
        const uint64_t rlo = fs + (uint64_t)tp0 * Bf;
        const uint64_t rhi = fs + (uint64_t)tp1 * Bf;
        const uint64_t cend = rhi < b1 ? rhi : b1;
        if (cend > pos) {
          const uint32_t code = a.rec.code[j];
          const int s = code & 0xff, ss = (code >> 8) & 0xff, ds = (code >> 16) & 0xff,
                    ts = code >> 24;
          const uint64_t u0 = pos - rlo;
          const int64_t len = (int64_t)(cend - pos);
          const uint8_t* sp;
          uint8_t* dp[kMaxWorld];
          int R = 0;
          int64_t msg_field = 0;
          if (a.mode != kDirect) {
            const int key = ss * Sd + ds;
            const int64_t kt = h->key_tokens[key];
            int64_t fb = 0;
            for (int ff = 0; ff < f; ++ff) fb += (kt * a.Bf[ff] + 15) & ~15LL;
            msg_field = h->msg_off[key] + fb + a.rec.msg_tok[j] * (int64_t)Bf + (int64_t)u0;
          }
          if (a.mode == kUnpack) sp = a.stage[s] + msg_field;
          else sp = a.src[s][f] + a.rec.src_tok[j] * (int64_t)Bf + (int64_t)u0;
          if (a.mode == kPack) {
            dp[0] = a.stage[s] + msg_field;
            R = 1;
          } else {
            const int64_t doff = a.rec.dst_tok[j] * (int64_t)Bf + (int64_t)u0;
            for (int td = ts; td < a.tp_d; td += a.tp_s) {
              const int d = a.rank0_d + ds * a.tp_d + td;
              uint8_t* base = a.dst[d][f];
              if (base != nullptr) dp[R++] = base + doff;
            }
          }
          if (R > 0) warp_copy(sp, dp, R, len, lane);
          pos = cend;
        }
        if (pos >= rhi) {
          ++j;
          if (j == rend) { j = rbeg; ++f; }
        }
      }
    }
  }
  // completion (multi-process comm): last CTA releases this epoch to every peer and waits
  if (a.world > 1 && a.view_rank >= 0) {
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned prev = atomicAdd(a.done_ctr, 1u);
      s_last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (s_last && threadIdx.x < 32) {
      if (threadIdx.x == 0) *a.done_ctr = 0;
      __threadfence_system();
      const unsigned miss = signal_and_wait(a.my_pad, a.peer_pad, a.world, a.me, kDoneSlot,
                                            a.epoch, a.timeout_ns);
      if (threadIdx.x == 0 && miss) {
        if (atomicCAS(a.err, 0, EARL_ERR_TIMEOUT) == 0) *a.err_detail = (int32_t)miss;
      }
    }
  }
}

}  // namespace

cudaError_t launch_copy(const CopyArgs& a, int grid, int block, cudaStream_t s) {
  copy_kernel<<<grid, block, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_entry_barrier(uint64_t* my_pad, uint64_t* const* peer_pad, int world, int me,
                                 uint64_t epoch, uint64_t timeout_ns, int32_t* err,
                                 int32_t* err_detail, cudaStream_t s) {
  PeerPads pads;
  for (int p = 0; p < kMaxWorld; ++p) pads.p[p] = peer_pad[p];
  entry_barrier_kernel<<<1, 32, 0, s>>>(my_pad, pads, world, me, epoch, timeout_ns, err,
                                        err_detail);
  return cudaGetLastError();
}

}  // namespace earl
