// aggregate.cu -- NEXT-2 of SURVEY.md §8(f): distributed per-sequence aggregation before the
// dispatch ("rewards and returns are aggregated for advantage estimation.  We
// will improve this process in a distributed manner").
//
// On the ranks of the source layout (sequences whole: SP = 1), where the rollout produced them:
//   returns    G_t = m_t r_t + gamma G_{t+1} per sequence (G_L = 0)           -- returns_kernel
//              + fp64 partial sums (sum m, sum m G, sum m G^2) over replica-0 tokens
//   (all-reduce of the 3 partials across ranks by the caller: no controller)
//   advantages A_t = m_t (G_t - mu) / (sigma + eps), mu / sigma over the batch's masked tokens
//                                                                               -- advantage_kernel
// (REINFORCE++-style globally normalised returns; reading n5).  Both kernels are
// HBM-bound elementwise/scan work; no tensor cores.
//
// returns_kernel: one segmented backward scan over each rank's token buffer.  Token t carries
// the affine map x -> v_t + g_t x with v_t = m_t r_t and g_t = 0 if t is the last token of its
// sequence, else gamma; G_t is the composition of the maps of t..end applied to 0.  The buffer
// is cut into aligned windows of up to 4096 tokens; a warp claims windows right to left from
// an atomic counter and streams its window twice in 512-token batches (16 contiguous tokens
// per lane).  A batch arrives by two TMA bulk copies (rewards, mask) into a per-warp 2-slot
// shared-memory ring, one batch ahead, and lanes read their 16 tokens in a rotated,
// bank-conflict-free order (the kernel was L1-bound on lane-strided global loads): pass 1
// composes the window's map and publishes it, a lane-parallel look-back over the windows to its right stops at the first inclusive value or zero slope (a
// sequence end), pass 2 re-reads the window from L2 and writes G with float4 stores.  HBM sees
// every token read and written once; long sequences are spread over many warps (decoupled
// look-back).
#include <cooperative_groups.h>

#include "earl_internal.cuh"

namespace earl {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kTokLane = 16;              // contiguous tokens of a lane in a batch
constexpr int kBatch = 32 * kTokLane;     // 512 tokens per batch
#ifndef EARL_AGG_MAX_NB
#define EARL_AGG_MAX_NB 8
#endif
#ifndef EARL_AGG_PF
#define EARL_AGG_PF 0
#endif
constexpr int kMaxNB = EARL_AGG_MAX_NB;   // batches per window (at most)
constexpr int kMaxWin = kBatch * kMaxNB;  // 4096 tokens
constexpr int kWarps = 8;                 // warps per CTA
#ifndef EARL_AGG_CTAS_PER_SM
#define EARL_AGG_CTAS_PER_SM 3
#endif
constexpr int kCtasPerSm = EARL_AGG_CTAS_PER_SM;

__device__ __forceinline__ void latch(PlanHeader* h, int code, int detail) {
  if (atomicCAS(&h->err, 0, code) == 0) h->err_detail = detail;
}

// gate (AggArgs::gate) on the batch, read on the device: lets the host launch every returns
// kernel when it does not know the batch (all but the chosen one exit at once).  gate = id + 1
// runs kernel id (ReturnsKernel) only if choose_returns picks it.  Whole-CTA decision.
// Warp-collective (warp 0): lane r reads source rank r's token count, so the header costs one
// round trip (a loop in one thread had serialised them: ~1 us per rank at every launch).
__device__ int device_choice(const AggArgs& a, int* coop_nb) {
  const PlanHeader* h = a.hdr;
  const LayoutDesc& S = a.plan.lay[0];
  const int lane = threadIdx.x & 31;
  const int q = lane - S.rank0;
  const bool in = lane < a.world && (a.view_rank < 0 || lane == a.view_rank) && q >= 0 &&
                  q < S.dp * S.tp;
  const int64_t mine = in ? *reinterpret_cast<const volatile int64_t*>(&h->shard_tokens[0][q / S.tp]) : 0;
  const int64_t m = *reinterpret_cast<const volatile int64_t*>(&h->max_len);
  const unsigned mask = __ballot_sync(kFull, in);
  int64_t nt[kMaxWorld];
  int n = 0;
  for (int r = 0; r < kMaxWorld; ++r) {
    const int64_t v = __shfl_sync(kFull, mine, r);
    if (mask >> r & 1u) nt[n++] = v;
  }
  return choose_returns(nt, n, m, a.resident_warps, a.coop_warps, coop_nb);
}

__device__ bool gated_out(const AggArgs& a) {
  if (a.gate == 0) return false;
  __shared__ int s_out;
  if (threadIdx.x < 32) {
    const int c = device_choice(a, nullptr);
    if (threadIdx.x == 0) s_out = c != a.gate - 1;
  }
  __syncthreads();
  return s_out != 0;
}

__device__ __forceinline__ uint64_t ld_word(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_word(uint64_t* p, uint32_t tag, float x) {
  const uint64_t v = ((uint64_t)tag << 32) | __float_as_uint(x);
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ bool word_is(uint64_t w, uint32_t tag) { return (uint32_t)(w >> 32) == tag; }
__device__ __forceinline__ float word_val(uint64_t w) { return __uint_as_float((uint32_t)w); }

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// L2 prefetch of batch b of a window (token bytes, then mask bytes): lanes 0..15 take the 16
// lines of rewards, lanes 16..19 the 4 lines of mask
__device__ __forceinline__ void prefetch_batch(const float* rw, const uint8_t* mk, int64_t t0,
                                               int64_t w1, int lane) {
  if (lane < 16) {
    const int64_t t = t0 + 32 * lane;
    if (t < w1) prefetch_l2(rw + t);
  } else if (lane < 20) {
    const int64_t t = t0 + 128 * (lane - 16);
    if (t < w1) prefetch_l2(mk + t);
  }
}

__device__ __forceinline__ bool aligned(const void* p, unsigned a) {
  return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0;
}

// Source ranks of the launch (SP = 1: rank = rank0 + g*TP + t holds group g whole).
struct RankTable {
  int n;
  int nb;                           // batches per window of this launch
  int rank[kMaxWorld];
  int t[kMaxWorld];
  int64_t gs[kMaxWorld];            // first sorted position of the rank's group
  int64_t cnt[kMaxWorld];           // sequences of the rank
  int64_t ntok[kMaxWorld];          // tokens of the rank
  int64_t wbeg[kMaxWorld + 1];      // first window (work unit) of the rank
};

// The window size adapts to the batch: 4096 tokens once there are two windows per warp of
// the grid, down to one 512-token batch for small batches (every warp busy, short chains).
// Warp-collective (warp 0): lane r reads source rank r's header fields, one round trip.
__device__ void rank_table(const AggArgs& a, RankTable& rt, int64_t warps, int nb_fixed = 0) {
  const PlanHeader* h = a.hdr;
  const LayoutDesc& S = a.plan.lay[0];
  const int lane = threadIdx.x & 31;
  const int q = lane - S.rank0;
  const bool in = lane < a.world && (a.view_rank < 0 || lane == a.view_rank) && q >= 0 &&
                  q < S.dp * S.tp;
  const unsigned mask = __ballot_sync(kFull, in);
  const int idx = __popc(mask & ((1u << lane) - 1u));
  int64_t nt = 0;
  if (in) {
    const int g = q / S.tp;
    rt.rank[idx] = lane;
    rt.t[idx] = q % S.tp;
    rt.gs[idx] = h->group_start[0][g];
    rt.cnt[idx] = h->group_count[0][g];
    nt = h->shard_tokens[0][g];
    rt.ntok[idx] = nt;
  }
  int64_t batches = (nt + kBatch - 1) / kBatch;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) batches += __shfl_xor_sync(kFull, batches, o);
  const int n = __popc(mask);
  const int nb = nb_fixed > 0 ? nb_fixed : (int)max((int64_t)1, min((int64_t)kMaxNB, batches / (2 * warps)));
  const int64_t win = (int64_t)kBatch * nb;
  // window prefix in rank order (idx grows with the lane among the ranks taking part)
  const int64_t cnt = in ? (nt + win - 1) / win : 0;
  int64_t inc = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(kFull, inc, o);
    if (lane >= o) inc += y;
  }
  if (in) rt.wbeg[idx] = inc - cnt;
  const int64_t all = __shfl_sync(kFull, inc, 31);
  if (lane == 0) {
    rt.n = n;
    rt.nb = nb;
    rt.wbeg[n] = all;
    if (n == 0) rt.wbeg[0] = 0;
  }
  __syncwarp();
}

// Smallest p in [lo, hi] with cum[p] - base >= key (cum[hi] - base >= key holds): 32-ary
// warp search, one gather per level.
__device__ int64_t first_at_least(const int64_t* cum, int64_t base, int64_t lo, int64_t hi,
                                  int64_t key, int lane) {
  while (hi - lo >= 32) {
    const int64_t step = (hi - lo + 31) / 32;
    int64_t p = lo + (int64_t)lane * step;
    if (p > hi) p = hi;
    const unsigned b = __ballot_sync(kFull, cum[p] - base >= key);
    if (b == 0) {
      lo = lo + 31 * step + 1;
    } else {
      const int f = __ffs(b) - 1;
      const int64_t pf = min(lo + (int64_t)f * step, hi);
      lo = f ? lo + (int64_t)(f - 1) * step + 1 : lo;
      hi = pf;
    }
  }
  const int64_t p = lo + lane;
  const unsigned b = __ballot_sync(kFull, p <= hi && cum[min(p, hi)] - base >= key);
  return lo + (__ffs(b) - 1);
}

// Sequence ends inside the window [w0, w1): bit (s-1-w0) of bm for every sequence start s in
// (w0, w1] (starts are cum[p] - base, p in [gs, pend]; the last one ends the buffer).  Clears
// the window's nwords words first; returns the first sequence p with cum[p] - base >= w0.
__device__ __forceinline__ int64_t mark_ends(uint32_t* bm, int nwords, const int64_t* cum,
                                             int64_t base, int64_t gs, int64_t pend, int64_t w0,
                                             int64_t w1, int lane) {
  for (int j = lane; j < nwords; j += 32) bm[j] = 0u;
  __syncwarp();
  const int64_t lo = first_at_least(cum, base, gs, pend, w0, lane);
  for (int64_t p0 = lo;; p0 += 32) {
    const int64_t p = p0 + lane;
    const int64_t s = p <= pend ? cum[p] - base : INT64_MAX;
    const bool in = s <= w1;
    if (in && s > w0) atomicOr(&bm[(s - 1 - w0) >> 5], 1u << ((s - 1 - w0) & 31));
    if (__ballot_sync(kFull, in) != kFull) break;
  }
  __syncwarp();
  return lo;
}

// In-order composition of the 32 lane maps (lane l's map applies after lane l+1's):
// (rS, rP) = exclusive suffix (lanes right of this one), (tS, tP) = all 32 lanes.
__device__ __forceinline__ void warp_compose(float S, float P, int lane, float& rS, float& rP,
                                             float& tS, float& tP) {
  float sS = S, sP = P;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const float oS = __shfl_down_sync(kFull, sS, off), oP = __shfl_down_sync(kFull, sP, off);
    if (lane + off < 32) { sS = sS + sP * oS; sP = sP * oP; }
  }
  rS = __shfl_down_sync(kFull, sS, 1);
  rP = __shfl_down_sync(kFull, sP, 1);
  if (lane == 31) { rS = 0.f; rP = 1.f; }
  tS = __shfl_sync(kFull, sS, 0);
  tP = __shfl_sync(kFull, sP, 0);
}

// A lane's 16 tokens of a batch.  Tokens past the buffer load as r = 0, m = 0: they add nothing
// and sit right of the buffer's last token, which ends its sequence, so their slopes are moot.
struct Batch {
  float4 r[4];
  uint4 m;  // the 16 mask bytes
};

// unaligned buffers or the rank's tail: token by token (rare; a rolled loop keeps it small)
__device__ __forceinline__ void load_batch_scalar(Batch& B, const float* rw, const uint8_t* mk,
                                                  int64_t t, int64_t w1) {
  float x[kTokLane];
  uint32_t m[4] = {0u, 0u, 0u, 0u};
#pragma unroll 1
  for (int i = 0; i < kTokLane; ++i) {
    x[i] = 0.f;
    if (t + i < w1) {
      x[i] = rw[t + i];
      m[i >> 2] |= (uint32_t)mk[t + i] << (8 * (i & 3));
    }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) B.r[k] = make_float4(x[4 * k], x[4 * k + 1], x[4 * k + 2], x[4 * k + 3]);
  B.m = make_uint4(m[0], m[1], m[2], m[3]);
}

template <bool kLastUse>
__device__ __forceinline__ void load_batch(Batch& B, const float* rw, const uint8_t* mk, int64_t t,
                                           int64_t w1, bool vec) {
  if (vec && t + kTokLane <= w1) {
    const float4* rp = reinterpret_cast<const float4*>(rw + t);
    const uint4* mp = reinterpret_cast<const uint4*>(mk + t);
#pragma unroll
    for (int k = 0; k < 4; ++k) B.r[k] = kLastUse ? __ldcs(rp + k) : __ldca(rp + k);
    B.m = kLastUse ? __ldcs(mp) : __ldca(mp);
  } else {
    load_batch_scalar(B, rw, mk, t, w1);
  }
}

// token i of the lane's 16 is masked in: its mask byte is nonzero (boolean mask, reading n5);
// one LOP3 with a byte-wide immediate per token
__device__ __forceinline__ bool tok_on(const Batch& B, int i) {
  const int k = i >> 2;
  const uint32_t w = k == 0 ? B.m.x : k == 1 ? B.m.y : k == 2 ? B.m.z : B.m.w;
  return (w & (0xffu << (8 * (i & 3)))) != 0u;
}

__device__ __forceinline__ float tok_r(const Batch& B, int i) {
  const float4& v = B.r[i >> 2];
  const int c = i & 3;
  return c == 0 ? v.x : c == 1 ? v.y : c == 2 ? v.z : v.w;
}

#ifndef EARL_AGG_TMA
#define EARL_AGG_TMA 1  // batches arrive by TMA bulk copies (0: register loads, lane-contiguous)
#endif
#ifndef EARL_AGG_SLOTS
#define EARL_AGG_SLOTS 2
#endif
constexpr int kSlots = EARL_AGG_SLOTS;  // batches in a warp's ring (kSlots - 1 loads ahead)
constexpr int kSlotBytes = kBatch * 4 + kBatch;  // a batch's rewards, then its mask bytes

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Per-warp 2-slot ring of whole batches loaded by TMA bulk copies (no LSU wavefronts on the
// global side).  Slot uses alternate; every use completes one phase of the slot's mbarrier (a
// batch that is not whole and 16-B aligned arrives without a copy and is read from global).
struct BatchRing {
  uint8_t* mem;       // this warp's kSlots slots
  uint64_t* bar;      // this warp's kSlots mbarriers
  uint32_t issued, got;
  bool tma[kSlots];

  __device__ __forceinline__ void init(uint8_t* m, uint64_t* b, int lane) {
    mem = m; bar = b; issued = got = 0;
    for (int s = 0; s < kSlots; ++s) tma[s] = false;
    if (lane == 0) {
      for (int s = 0; s < kSlots; ++s)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bar[s])) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
  }
  // start loading batch [t0, t0 + kBatch) into the next slot (its previous batch is consumed)
  __device__ __forceinline__ void issue(const float* rw, const uint8_t* mk, int64_t t0, int64_t w1,
                                        bool vec, int lane) {
    const int s = issued % kSlots;
    const bool whole = vec && t0 + kBatch <= w1;
    tma[s] = whole;
    __syncwarp();
    if (lane == 0) {
      const uint32_t b = smem_addr(&bar[s]);
      if (whole) {
        uint8_t* dst = mem + s * kSlotBytes;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b),
                     "r"((uint32_t)kSlotBytes) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(smem_addr(dst)), "l"(rw + t0), "r"((uint32_t)(kBatch * 4)), "r"(b) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(smem_addr(dst + kBatch * 4)), "l"(mk + t0), "r"((uint32_t)kBatch), "r"(b)
            : "memory");
      } else {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
      }
    }
    ++issued;
  }
  // this lane's 16 tokens of the oldest issued batch (its lane tokens start at t)
  template <bool kLastUse>
  __device__ __forceinline__ void get(Batch& B, const float* rw, const uint8_t* mk, int64_t t,
                                      int64_t w1, bool vec, int lane) {
    const int s = got % kSlots;
    const uint32_t parity = (got / kSlots) & 1;
    const uint32_t b = smem_addr(&bar[s]);
    uint32_t done;
    do {
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
          " selp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done) : "r"(b), "r"(parity) : "memory");
    } while (!done);
    ++got;
    if (!tma[s]) {
      load_batch<kLastUse>(B, rw, mk, t, w1, vec);
      return;
    }
    // rotated chunk order: lanes 2j, 2j+1 of a quarter-warp start at chunk j, so the 8
    // 16-B reads of a phase hit 8 distinct bank groups (a lane's 64 B span 4 of them)
    const uint8_t* rb = mem + s * kSlotBytes + 64 * lane;
    const int rot = (lane >> 1) & 3;
    float4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = *reinterpret_cast<const float4*>(rb + 16 * ((k + rot) & 3));
    // v[k] is chunk (k + rot) & 3: rotate so that B.r[c] = v[(c - rot) & 3]
    float4 u[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) u[c] = (rot & 1) ? v[(c + 3) & 3] : v[c];
#pragma unroll
    for (int c = 0; c < 4; ++c) B.r[c] = (rot & 2) ? u[(c + 2) & 3] : u[c];
    B.m = *reinterpret_cast<const uint4*>(mem + s * kSlotBytes + kBatch * 4 + 16 * lane);
  }
};

// Decoupled look-back for window w of a rank (windows w+1 .. nwin-1 lie to its right), 32
// windows per round trip: compose their maps up to the first inclusive value or zero slope (a
// sequence end); returns G just right of the window (0 past the buffer end).
__device__ __forceinline__ float look_back(AggWindow* W, int64_t w, int64_t nwin, uint32_t tag,
                                           int lane) {
  float cS = 0.f, cP = 1.f;
  for (int64_t j0 = w + 1; j0 < nwin;) {
    const int64_t j = j0 + lane;
    bool ready = false, stop = false;
    float S = 0.f, P = 1.f;
    if (j < nwin) {
      const uint64_t wi = ld_word(&W[j].inc);
      if (word_is(wi, tag | 2u)) {
        ready = stop = true;
        S = word_val(wi);
        P = 0.f;
      } else {
        const uint64_t ws = ld_word(&W[j].S), wp = ld_word(&W[j].P);
        if (word_is(ws, tag | 1u) && word_is(wp, tag | 1u)) {
          ready = true;
          S = word_val(ws);
          P = word_val(wp);
          stop = P == 0.f;
        }
      }
    }
    // usable prefix: ready lanes up to (and including) the first stopper
    const unsigned rmask = __ballot_sync(kFull, ready);
    const unsigned smask = __ballot_sync(kFull, stop);
    const int n_ready = (~rmask) ? __ffs(~rmask) - 1 : 32;
    const int first_stop = smask ? __ffs(smask) - 1 : 32;
    const int n_use = min(n_ready, first_stop + 1);
    if (n_use == 0) { __nanosleep(32); continue; }
    if (lane >= n_use) { S = 0.f; P = 1.f; }
    float rS, rP, tS, tP;
    warp_compose(S, P, lane, rS, rP, tS, tP);
    cS = cS + cP * tS;
    cP = cP * tP;
    if (cP == 0.f || first_stop < n_use) break;
    j0 += n_use;
  }
  return cS;
}

// Per-sequence return G_0 of the sequences starting in the window [.., w1) (from sequence lo
// on; zero-length sequences at the buffer end belong to the last window).  G was written by this
// warp: the caller's __syncwarp orders the reads after it.
__device__ __forceinline__ void seq_returns(float* SR, const float* G, const int64_t* cum,
                                            int64_t base, int64_t gs, int64_t pend, int64_t lo,
                                            int64_t w1, int64_t ntok, int lane) {
  if (SR == nullptr) return;
  __syncwarp();
  for (int64_t p0 = lo;; p0 += 32) {
    const int64_t p = p0 + lane;
    bool in = false;
    if (p < pend) {
      const int64_t s = cum[p] - base;
      const int64_t L = cum[p + 1] - base - s;
      in = s < w1 || (s == w1 && w1 == ntok);
      if (in) SR[p - gs] = L > 0 ? G[s] : 0.f;
    }
    if (__ballot_sync(kFull, in) != kFull) break;
  }
}

// The end of returns_kernel: zero-length ranks' sequence returns, the block's fp64
// partials (one atomic per block), and the last CTA's reset of the claim counter + epoch.
__device__ __forceinline__ void returns_epilogue(const AggArgs& a, const RankTable& rt,
                                                 double (*red)[32], double s_m, double s_g,
                                                 double s_g2, int nwarps) {
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  // ranks without tokens still owe their (zero-length) sequences a return
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    for (int ri = 0; ri < rt.n; ++ri) {
      float* SR = a.seq_return[rt.rank[ri]];
      if (SR == nullptr || rt.ntok[ri] != 0) continue;
      for (int64_t j = lane; j < rt.cnt[ri]; j += 32) SR[j] = 0.f;
    }
  }

  // warp, then block reduction of the fp64 partials; one atomic per block
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    s_m += __shfl_xor_sync(kFull, s_m, off);
    s_g += __shfl_xor_sync(kFull, s_g, off);
    s_g2 += __shfl_xor_sync(kFull, s_g2, off);
  }
  if (lane == 0) { red[0][wid] = s_m; red[1][wid] = s_g; red[2][wid] = s_g2; }
  __syncthreads();
  if (threadIdx.x < 3) {
    double acc = 0.0;
    for (int k = 0; k < nwarps; ++k) acc += red[threadIdx.x][k];
    if (acc != 0.0) atomicAdd(a.partial + threadIdx.x, acc);
  }
  // the last CTA out resets the claim counter and advances the epoch (no host reset between
  // launches or graph replays)
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&a.ws->fin_ctr, 1u) == gridDim.x - 1) {
      a.ws->work_ctr = 0;
      a.ws->fin_ctr = 0;
      a.ws->epoch = a.ws->epoch + 1u;
      __threadfence();
    }
  }
}

__global__ void __launch_bounds__(kWarps * 32, kCtasPerSm) returns_kernel(const __grid_constant__ AggArgs a) {
  if (gated_out(a)) return;
  __shared__ RankTable rt;
  __shared__ uint32_t ends_bm[kWarps][kMaxWin / 32];
  __shared__ float2 bmap[kWarps][kMaxNB];   // per batch: its map (pass 1), then its carry
  __shared__ float2 lmap[kWarps][kMaxNB][32];  // per batch and lane: exclusive suffix map (pass 1)
  __shared__ double red[3][32];
  __shared__ uint32_t s_tag;
  __shared__ int s_ok;
#if EARL_AGG_TMA
  extern __shared__ __align__(128) uint8_t ring_mem[];  // [kWarps][kSlots][kSlotBytes]
  __shared__ uint64_t ring_bar[kWarps][kSlots];
#endif
  if (threadIdx.x < 32) rank_table(a, rt, (int64_t)gridDim.x * kWarps);
  if (threadIdx.x == 0) {
    s_tag = (*(volatile uint32_t*)&a.ws->epoch + 1u) << 2;  // | 1 aggregate, | 2 inclusive
    s_ok = rt.wbeg[rt.n] <= a.win_cap;
    if (!s_ok && blockIdx.x == 0)
      latch(a.plan.hdr, EARL_ERR_CAPACITY, (int)min(rt.wbeg[rt.n], (int64_t)INT32_MAX));
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const uint32_t tag = s_tag;
  const int64_t total = s_ok ? rt.wbeg[rt.n] : 0;
  const int NB = rt.nb;
  const int64_t win = (int64_t)kBatch * NB;
  const float gamma = a.gamma;
  const float g16 = a.gamma16;  // the slope of a lane's 16 tokens without a sequence end
  uint32_t* bm = ends_bm[wid];
  float2* bmp = bmap[wid];
  float2 (*lmp)[32] = lmap[wid];
  double s_m = 0.0, s_g = 0.0, s_g2 = 0.0;
#if EARL_AGG_TMA
  BatchRing ring;
  ring.init(ring_mem + (size_t)wid * kSlots * kSlotBytes, ring_bar[wid], lane);
#endif

  // windows are claimed in increasing order and every window only waits on smaller ones (no
  // deadlock); a warp claims its next window only when it starts it, so a window's right
  // neighbour is always already in progress (claiming ahead would make the left neighbour wait
  // a whole window for it)
  while (true) {
    uint32_t claim = 0;
    if (lane == 0) claim = atomicAdd(&a.ws->work_ctr, 1u);
    const int64_t u = __shfl_sync(kFull, claim, 0);
    if (u >= total) break;
    int ri = 0;
    while (u >= rt.wbeg[ri + 1]) ++ri;
    const int r = rt.rank[ri];
    const int64_t nwin = rt.wbeg[ri + 1] - rt.wbeg[ri];
    const int64_t w = nwin - 1 - (u - rt.wbeg[ri]);  // right to left within the rank
    const int64_t w0 = w * win;
    const int64_t w1 = min(rt.ntok[ri], w0 + win);
    const int nb = (int)((w1 - w0 + kBatch - 1) / kBatch);
    const float* rw = a.rewards[r];
    const uint8_t* mk = a.mask[r];
    float* G = a.returns[r];
    const bool vec = aligned(rw, 16) && aligned(G, 16) && aligned(mk, 16);
    const int64_t lt = w0 + (int64_t)kTokLane * lane;  // this lane's tokens in batch b: lt + 512 b

#if EARL_AGG_TMA
    Batch cur;
    for (int d = 1; d < kSlots && nb - d >= 0; ++d)
      ring.issue(rw, mk, w0 + (int64_t)(nb - d) * kBatch, w1, vec, lane);
#else
    Batch cur, nxt;  // batch b, and b-1 in flight
    load_batch<false>(cur, rw, mk, lt + (int64_t)(nb - 1) * kBatch, w1, vec);
#endif
    for (int d = 3; d < 3 + EARL_AGG_PF; ++d)
      if (nb >= d) prefetch_batch(rw, mk, w0 + (int64_t)(nb - d) * kBatch, w1, lane);

    // sequence ends inside the window: token s-1 for every sequence start s in (w0, w1]
    // (starts are cum[0][p] - cum[0][gs], p in [gs, gs+cnt]; the last one ends the buffer)
    const int64_t* cum = a.plan.cum[0];
    const int64_t gs = rt.gs[ri], pend = gs + rt.cnt[ri];
    const int64_t base = cum[gs];
    const int64_t lo = mark_ends(bm, nb * (kBatch / 32), cum, base, gs, pend, w0, w1, lane);
    // bit i: token i of this lane's 16 in batch b ends its sequence
    auto ends16 = [&](int b) { return (bm[16 * b + (lane >> 1)] >> (16 * (lane & 1))) & 0xffffu; };

    // pass 1: lane maps and batch maps (shared memory) and the window's map
    float wS = 0.f, wP = 1.f;
#pragma unroll 1
    for (int b = nb - 1; b >= 0; --b) {
#if EARL_AGG_TMA
      if (b - (kSlots - 1) >= 0)
        ring.issue(rw, mk, w0 + (int64_t)(b - (kSlots - 1)) * kBatch, w1, vec, lane);
      ring.get<false>(cur, rw, mk, lt + (int64_t)b * kBatch, w1, vec, lane);
#else
      if (b > 0) load_batch<false>(nxt, rw, mk, lt + (int64_t)(b - 1) * kBatch, w1, vec);
#endif
      if (EARL_AGG_PF > 0 && b >= 1 + EARL_AGG_PF)
        prefetch_batch(rw, mk, w0 + (int64_t)(b - 1 - EARL_AGG_PF) * kBatch, w1, lane);
      const uint32_t e = ends16(b);
      float S = 0.f;
#pragma unroll
      for (int i = kTokLane - 1; i >= 0; --i) {
        const float v = tok_on(cur, i) ? tok_r(cur, i) : 0.f;
        S = fmaf(((e >> i) & 1u) ? 0.f : gamma, S, v);
      }
      float rS, rP, bS, bP;
      warp_compose(S, e ? 0.f : g16, lane, rS, rP, bS, bP);
      lmp[b][lane] = make_float2(rS, rP);
      if (lane == 0) bmp[b] = make_float2(bS, bP);
      wS = bS + bP * wS;
      wP = bP * wP;
#if !EARL_AGG_TMA
      cur = nxt;
#endif
    }

    // publish the window's map, then look back (32 windows per round trip) for the carry:
    // compose the maps of windows w+1, w+2, ... up to the first inclusive value or zero slope
    AggWindow* W = a.win + rt.wbeg[ri];
    delay_inject(4 + (uint32_t)w);
    if (lane == 0 && w + 1 < nwin) {
      st_word(&W[w].S, tag | 1u, wS);
      st_word(&W[w].P, tag | 1u, wP);
    }
    delay_inject(5 + (uint32_t)w);
    const float carry = look_back(W, w, nwin, tag, lane);  // past the buffer end: G = 0
    if (lane == 0) {
      st_word(&W[w].inc, tag | 2u, wS + wP * carry);
      float c = carry;  // carries into the batches, right to left
      for (int b = nb - 1; b >= 0; --b) {
        const float2 m = bmp[b];
        bmp[b] = make_float2(c, 0.f);
        c = m.x + m.y * c;
      }
    }
    __syncwarp();

    // pass 2: returns from the lane maps and batch carries (the window's second read hits L2),
    // float4 stores, statistics
    const bool count_stats = rt.t[ri] == 0;
#if EARL_AGG_TMA
    for (int d = 1; d < kSlots && nb - d >= 0; ++d)
      ring.issue(rw, mk, w0 + (int64_t)(nb - d) * kBatch, w1, vec, lane);
#else
    load_batch<true>(cur, rw, mk, lt + (int64_t)(nb - 1) * kBatch, w1, vec);
#endif
#pragma unroll 1
    for (int b = nb - 1; b >= 0; --b) {
#if EARL_AGG_TMA
      if (b - (kSlots - 1) >= 0)
        ring.issue(rw, mk, w0 + (int64_t)(b - (kSlots - 1)) * kBatch, w1, vec, lane);
      ring.get<true>(cur, rw, mk, lt + (int64_t)b * kBatch, w1, vec, lane);
#else
      if (b > 0) load_batch<true>(nxt, rw, mk, lt + (int64_t)(b - 1) * kBatch, w1, vec);
#endif
      const uint32_t e = ends16(b);
      const float2 rm = lmp[b][lane];
      float g_next = rm.x + rm.y * bmp[b].x;
      float out[kTokLane];
#pragma unroll
      for (int i = kTokLane - 1; i >= 0; --i) {
        const float v = tok_on(cur, i) ? tok_r(cur, i) : 0.f;
        out[i] = fmaf(((e >> i) & 1u) ? 0.f : gamma, g_next, v);
        g_next = out[i];
      }
      if (count_stats) {
        float sg = 0.f, sg2 = 0.f;
        int cnt = 0;
#pragma unroll
        for (int i = 0; i < kTokLane; ++i) {
          if (tok_on(cur, i)) {
            sg += out[i];
            sg2 = fmaf(out[i], out[i], sg2);
            ++cnt;
          }
        }
        s_m += (double)cnt;
        s_g += (double)sg;
        s_g2 += (double)sg2;
      }
      const int64_t t = lt + (int64_t)b * kBatch;
      if (vec && t + kTokLane <= w1) {
        float4* gp = reinterpret_cast<float4*>(G + t);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          __stcs(gp + k, make_float4(out[4 * k], out[4 * k + 1], out[4 * k + 2], out[4 * k + 3]));
      } else {
        for (int i = 0; i < kTokLane; ++i)
          if (t + i < w1) G[t + i] = out[i];
      }
#if !EARL_AGG_TMA
      cur = nxt;
#endif
    }

    // per-sequence return G_0 of the sequences starting in the window (zero-length sequences
    // at the buffer end belong to the last window)
    seq_returns(a.seq_return[r], G, cum, base, gs, pend, lo, w1, rt.ntok[ri], lane);
    __syncwarp();
  }

  returns_epilogue(a, rt, red, s_m, s_g, s_g2, kWarps);
}

// ---------------------------------------------------------------------------------------
// returns_units_kernel: single pass, no look-back.  A unit is the run of whole sequences that
// start in [k * kUnitTok, (k+1) * kUnitTok) of a rank's buffer (the last unit also takes the
// trailing zero-length ones), so no return crosses a unit boundary: a warp claims a unit and
// streams it right to left in 512-token batches through a 3-slot TMA ring (2 batches ahead),
// composing each batch's lane maps and applying the carry from the batch to its right in
// registers -- every token read once from HBM and written once, no second pass, no published
// window maps.  The unit -> first sequence table comes from unit_table_kernel (one pass over the
// sequences).  Used when the batch's longest sequence is known to be <= kUnitMaxLen (a longer one
// would be streamed by a single warp); otherwise returns_kernel.
// ---------------------------------------------------------------------------------------

#ifndef EARL_AGG_USLOTS
#define EARL_AGG_USLOTS 3
#endif
constexpr int kUSlots = EARL_AGG_USLOTS;

// this lane's 16 tokens [t, t+16) restricted to [lo, hi): vector loads when whole and aligned
__device__ __forceinline__ void load_batch_in(Batch& B, const float* rw, const uint8_t* mk, int64_t t,
                                              int64_t lo, int64_t hi, bool vec) {
  if (vec && t >= lo && t + kTokLane <= hi) {
    const float4* rp = reinterpret_cast<const float4*>(rw + t);
    const uint4* mp = reinterpret_cast<const uint4*>(mk + t);
#pragma unroll
    for (int k = 0; k < 4; ++k) B.r[k] = __ldcs(rp + k);
    B.m = __ldcs(mp);
    return;
  }
  // fully unrolled, predicated: the 32 loads issue back to back (a rolled loop through a local
  // array serialised them, ~one memory latency per token)
  float x[kTokLane];
  uint32_t m[4] = {0u, 0u, 0u, 0u};
#pragma unroll
  for (int i = 0; i < kTokLane; ++i) {
    const bool in = t + i >= lo && t + i < hi;
    x[i] = in ? rw[t + i] : 0.f;
    m[i >> 2] |= (in ? (uint32_t)mk[t + i] : 0u) << (8 * (i & 3));
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) B.r[k] = make_float4(x[4 * k], x[4 * k + 1], x[4 * k + 2], x[4 * k + 3]);
  B.m = make_uint4(m[0], m[1], m[2], m[3]);
}

// bit k (k < 4) set for every nonzero byte k of w (mask bytes: any nonzero byte is 1, reading n5)
__device__ __forceinline__ uint32_t nonzero_bytes4(uint32_t w) {
  const uint32_t nz = (((w & 0x7f7f7f7fu) + 0x7f7f7f7fu) | w) & 0x80808080u;
  return (nz * 0x00204081u) >> 28;  // bytes' high bits 7, 15, 23, 31 -> bits 28..31
}

// unit -> first sequence (sorted position p in [gs, pend]) of every unit of every source rank of
// the launch: unit k of a rank starts at the first sequence whose start is >= k * kUnitTok.
__global__ void unit_table_kernel(const __grid_constant__ AggArgs a) {
  if (gated_out(a)) return;
  __shared__ RankTable rt;
  if (threadIdx.x < 32) rank_table(a, rt, 1, kUnitTok / kBatch);
  __syncthreads();
  if (rt.wbeg[rt.n] > a.win_cap) return;  // the unit kernel latches CAPACITY
  const int64_t* cum = a.plan.cum[0];
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  // one flat pass over every rank's positions gs .. pend (a loop per rank had put one HBM round
  // trip per rank on the critical path)
  int64_t pre[kMaxWorld + 1];
  pre[0] = 0;
  for (int ri = 0; ri < rt.n; ++ri)
    pre[ri + 1] = pre[ri] + (rt.wbeg[ri + 1] > rt.wbeg[ri] ? rt.cnt[ri] + 1 : 0);
  for (int64_t x = tid; x < pre[rt.n]; x += nth) {
    int ri = 0;
    while (x >= pre[ri + 1]) ++ri;
    const int64_t gs = rt.gs[ri], pend = gs + rt.cnt[ri], nu = rt.wbeg[ri + 1] - rt.wbeg[ri];
    const int64_t p = gs + (x - pre[ri]);
    const int64_t base = cum[gs];
    int64_t* tab = a.unit_first + rt.wbeg[ri];
    const int64_t s = cum[p] - base;                   // start of sequence p (ntok for pend)
    const int64_t kl = p == gs ? 0 : (cum[p - 1] - base) / kUnitTok + 1;
    int64_t kh = s / kUnitTok;
    if (p == pend || kh > nu - 1) kh = nu - 1;
    for (int64_t k = kl; k <= kh; ++k) tab[k] = p;
  }
}

// per-sequence return G_0 of sequences [p0, p1) (written by this warp: the caller syncs)
__device__ __forceinline__ void unit_seq_returns(float* SR, const float* G, const int64_t* cum,
                                                 int64_t base, int64_t gs, int64_t p0, int64_t p1,
                                                 int lane) {
  if (SR == nullptr) return;
  for (int64_t p = p0 + lane; p < p1; p += 32) {
    const int64_t s = cum[p] - base;
    const int64_t L = cum[p + 1] - base - s;
    SR[p - gs] = L > 0 ? G[s] : 0.f;
  }
}

// ---------------------------------------------------------------------------------------
// The per-batch path is kept lean (an earlier version spent ~670 warp instructions per batch,
// two thirds of them outside the recurrence, by ncu's source counters):
//  * lane 0 alone produces: it claims units into a per-warp queue in shared memory (skipping
//    units that hold no sequence), tracks its own issue cursor and issues the TMA copies; the
//    other lanes never execute producer code;
//  * no per-slot flags: producer and consumer derive "this batch came by TMA" from the batch's
//    range (vec, unit bounds, buffer end), so nothing lives in local memory;
//  * sequence ends come from a register window of the unit's sequence starts (lane j holds the
//    j-th start from the right; one ballot per batch, a shuffle per end), not from a shared-memory
//    bitmap rebuilt every 8 batches;
//  * a batch fully inside its unit with no sequence end takes a path with constant slopes: the
//    lane composition shuffles S only (the slopes are gamma^(16 * 2^k) and gamma^(16 * (31 - l)),
//    per-lane constants), no per-token slope selects, no unit-bound masks;
//  * the next unit's sequence starts are loaded while the current unit runs (the load's latency
//    hides behind its batches), and per-sequence returns come from that window too.
// ---------------------------------------------------------------------------------------

#ifndef EARL_AGG_UQ
#define EARL_AGG_UQ 8
#endif
constexpr int kUQ = EARL_AGG_UQ;  // claimed units queued per warp (power of two)
#ifndef EARL_AGG_U2CTAS
#define EARL_AGG_U2CTAS 2
#endif
constexpr int kU2Ctas = EARL_AGG_U2CTAS;  // CTAs per SM (8 warps each)

struct UnitQ {
  int64_t base;       // cum[gs] of the rank + ua: the unit's first token as a global prefix
  int32_t p0, p1;     // sequences [p0, p1) (sorted positions)
  int32_t ua, ub;     // the unit's tokens [ua, ub) of the rank buffer
  int32_t ri;         // rank index in the RankTable; -1: no more units
  int32_t pad;
};

constexpr int kNoStart = INT32_MIN / 2;  // an empty window entry (left of every batch)

// Positions inside a rank buffer are int32 here: the kernel refuses (CAPACITY) a rank of more
// than kU2MaxTok tokens, and prefer_units never picks it for one.
__global__ void __launch_bounds__(kWarps * 32, kU2Ctas) returns_units_kernel(const __grid_constant__ AggArgs a) {
  __shared__ RankTable rt;
  __shared__ double red[3][32];
  extern __shared__ __align__(128) uint8_t uring_mem[];  // [kWarps][kUSlots][kSlotBytes]
  __shared__ uint64_t uring_bar[kWarps][kUSlots];
  __shared__ UnitQ s_q[kWarps][kUQ];
  __shared__ int s_ok;
  if (gated_out(a)) return;
  if (threadIdx.x < 32) rank_table(a, rt, 1, kUnitTok / kBatch);
  if (threadIdx.x == 0) {
    bool ok = rt.wbeg[rt.n] <= a.win_cap;
    int64_t big = 0;
    for (int ri = 0; ri < rt.n; ++ri) big = max(big, rt.ntok[ri]);
    s_ok = ok && big <= kU2MaxTok;
    if (!s_ok && blockIdx.x == 0)
      latch(a.plan.hdr, EARL_ERR_CAPACITY, (int)min(ok ? big : rt.wbeg[rt.n], (int64_t)INT32_MAX));
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const uint32_t total = s_ok ? (uint32_t)rt.wbeg[rt.n] : 0u;
  const int64_t* cum = a.plan.cum[0];
  const float gamma = a.gamma;
  // slopes of the constant-slope path (kernel parameters: constant-bank operands):
  // a.gpw[k] = gamma^(16 * 2^k) (a run of 2^k lanes), a.g4 (a 4-token chunk), a.g512 (a batch);
  // rPl = gamma^(16 * (31 - lane)) (the lanes right of this one)
  float rPl = 1.f;
#pragma unroll
  for (int k = 0; k < 5; ++k)
    if (((31 - lane) >> k) & 1) rPl *= a.gpw[k];
  const int rot = (lane >> 1) & 3;  // ring read order: lanes 2j, 2j+1 of a quarter-warp start at chunk j

  uint8_t* ring = uring_mem + (size_t)wid * kUSlots * kSlotBytes;
  uint64_t* bar = uring_bar[wid];
  UnitQ* q = s_q[wid];
  if (lane == 0) {
    for (int s = 0; s < kUSlots; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bar[s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  // ---- producer state (lane 0 only) ----
  int p_nclaim = 0;        // units queued so far
  int p_iu = -1;           // queue index of the unit being issued
  int p_pb = 0, p_pbf = 1; // next batch to issue (descending) and the unit's first batch
  int p_ua = 0, p_ub = 0, p_ntok = 0;
  const float* p_rw = nullptr;
  const uint8_t* p_mk = nullptr;
  bool p_vec = false, p_done = false;
  uint32_t p_slot = 0;     // next ring slot to issue into
  uint32_t p_issued = 0;   // batches issued so far

  // lane 0: claim one unit with sequences into the queue (or an end marker)
  auto claim = [&]() {
    UnitQ& e = q[p_nclaim & (kUQ - 1)];
    for (;;) {
      delay_inject(8);
      const uint32_t u = atomicAdd(&a.ws->work_ctr, 1u);
      if (u >= total) { e.ri = -1; p_done = true; break; }
      int ri = 0;
      while (u >= (uint32_t)rt.wbeg[ri + 1]) ++ri;
      const int64_t gs = rt.gs[ri];
      const int64_t p0 = a.unit_first[u];
      const int64_t p1 = u + 1 < (uint32_t)rt.wbeg[ri + 1] ? a.unit_first[u + 1] : gs + rt.cnt[ri];
      if (p0 == p1) continue;  // no sequence starts in this unit's range
      const int64_t base = cum[gs], s0 = cum[p0], s1 = cum[p1];
      e.p0 = (int)p0; e.p1 = (int)p1; e.ri = ri;
      e.ua = (int)(s0 - base); e.ub = (int)(s1 - base);
      e.base = s0;
      break;
    }
    ++p_nclaim;
  };
  // lane 0: issue batches (right to left through the queued units) until kUSlots - 1 are in
  // flight beyond the c_n consumed, at most kUQ - 1 units ahead of the consumer's unit kc
  auto produce = [&](int kc, uint32_t c_n) {
    while (p_issued - c_n < (uint32_t)(kUSlots - 1)) {
      while (p_pb < p_pbf) {  // the unit being issued is done: move to the next one
        if (p_iu + 1 >= p_nclaim) {
          if (p_done || p_nclaim - kc >= kUQ - 1) return;
          claim();
          if (p_done) return;
        }
        ++p_iu;
        const UnitQ& e = q[p_iu & (kUQ - 1)];
        if (e.ri < 0) { p_pb = 0; p_pbf = 1; return; }  // the end marker
        const int r = rt.rank[e.ri];
        p_ua = e.ua; p_ub = e.ub; p_ntok = (int)rt.ntok[e.ri];
        p_rw = a.rewards[r]; p_mk = a.mask[r];
        p_vec = aligned(p_rw, 16) && aligned(p_mk, 16);
        p_pbf = p_ua / kBatch;
        p_pb = p_ua < p_ub ? (p_ub - 1) / kBatch : p_pbf - 1;  // no batches for an empty unit
      }
      const int t0 = p_pb * kBatch;
      const uint32_t b = smem_addr(&bar[p_slot]);
      // the batch's tokens inside the unit (rewards from a 4-token, the mask from a 16-token
      // granule); a whole batch inside the unit and the buffer is the common case
      bool ok = p_vec;
      int r0 = t0, m0 = t0;
      uint32_t rb = kBatch * 4, mb = kBatch;
      if (!(t0 >= p_ua && t0 + kBatch <= p_ub && t0 + kBatch <= p_ntok)) {
        const int lo = max(t0, p_ua), hi = min(t0 + kBatch, p_ub);
        const int m1 = (hi + 15) & ~15;
        ok = ok && m1 <= p_ntok;
        r0 = lo & ~3;
        m0 = lo & ~15;
        rb = (uint32_t)(((hi + 3) & ~3) - r0) * 4u;
        mb = (uint32_t)(m1 - m0);
      }
      if (ok) {
        const uint32_t dst = smem_addr(ring + p_slot * kSlotBytes);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(rb + mb) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(dst + (uint32_t)(r0 - t0) * 4u), "l"(p_rw + r0), "r"(rb), "r"(b) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(dst + kBatch * 4 + (uint32_t)(m0 - t0)), "l"(p_mk + m0), "r"(mb), "r"(b) : "memory");
      } else {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
      }
      p_slot = p_slot + 1 == kUSlots ? 0 : p_slot + 1;
      --p_pb;
      ++p_issued;
    }
  };

  if (lane == 0) {
    claim();
    produce(0, 0);
  }
  __syncwarp();

  // ---- consumer (every lane) ----
  double s_m = 0.0, s_g = 0.0, s_g2 = 0.0;
  uint32_t c_slot = 0, c_phase = 0;  // bit s: parity of slot s's next completion
  uint32_t c_n = 0;                  // batches consumed
  // sequence-start window of a unit: lane j holds the start of sequence top - j relative to the
  // unit (for top - j > p0), else kNoStart
  auto load_window = [&](const UnitQ& u, int top) -> int {
    const int p = top - lane;
    return p > u.p0 ? (int)(cum[p] - u.base) : kNoStart;
  };
  UnitQ cu = q[0];
  int ws = cu.ri >= 0 ? load_window(cu, cu.p1) : kNoStart;
  int nws = kNoStart;        // the next unit's window (loaded ahead)
  bool nx_loaded = false;
  for (int kc = 0; cu.ri >= 0; ++kc) {
    const int ri = cu.ri;
    const int r = rt.rank[ri];
    const int ua = cu.ua, ulen = cu.ub - cu.ua, ntok = (int)rt.ntok[ri];
    float* G = a.returns[r] + ua;            // the unit's tokens
    const float* rw = a.rewards[r];
    const uint8_t* mk = a.mask[r];
    const bool vec = aligned(rw, 16) && aligned(mk, 16);
    const bool vstore = aligned(a.returns[r], 16);  // G + lt = returns + t0 + 16 lane
    const bool count_stats = rt.t[ri] == 0;
    int wtop = cu.p1;          // sorted position of lane 0's window entry
    float carry = 0.f;         // G right of the current batch (the unit's last token ends a sequence)
    const int bf = ua / kBatch;
    const int bl = ulen > 0 ? (cu.ub - 1) / kBatch : bf - 1;
#pragma unroll 1
    for (int bb = bl; bb >= bf; --bb) {
      const int t0 = bb * kBatch;
      const int tb = t0 - ua;  // the batch's first token, relative to the unit
      // sequence ends in the batch: starts s with tb < s <= tb + kBatch end a sequence at s - 1
      uint32_t e = 0;
      for (;;) {
        unsigned bal = __ballot_sync(kFull, ws > tb && ws <= tb + kBatch);
        while (bal) {
          const int j = __ffs(bal) - 1;
          bal &= bal - 1;
          const int pos = __shfl_sync(kFull, ws, j) - 1 - tb;
          if ((pos >> 4) == lane) e |= 1u << (pos & 15);
        }
        const int last = __shfl_sync(kFull, ws, 31);
        if (last <= tb || wtop - 32 <= cu.p0) break;  // the window reaches left of the batch
        wtop -= 32;
        ws = load_window(cu, wtop);
      }
      // wait for the batch
      {
        const uint32_t b = smem_addr(&bar[c_slot]);
        const uint32_t parity = (c_phase >> c_slot) & 1u;
        uint32_t done;
        do {
          asm volatile(
              "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
              " selp.u32 %0, 1, 0, p;\n}\n"
              : "=r"(done) : "r"(b), "r"(parity) : "memory");
        } while (!done);
        c_phase ^= 1u << c_slot;
      }
      const int lo = max(t0, ua), hi = min(t0 + kBatch, cu.ub);
      const bool tma = vec && ((hi + 15) & ~15) <= ntok;
      const int lt = tb + kTokLane * lane;  // this lane's first token, relative to the unit
      // cur.r[k] = physical chunk k of the lane's 16 tokens = logical chunk (k + prot) & 3
      // (tokens 4c .. 4c+3): the ring is read in a rotated chunk order (conflict-free), and the
      // constant-slope path works in that order (chunk maps, no per-token de-rotation)
      Batch cur;
      int prot = 0;
      if (tma) {
        const uint8_t* rb = ring + c_slot * kSlotBytes + 64 * lane;
        prot = rot;
#pragma unroll
        for (int k = 0; k < 4; ++k) cur.r[k] = *reinterpret_cast<const float4*>(rb + 16 * ((k + rot) & 3));
        cur.m = *reinterpret_cast<const uint4*>(ring + c_slot * kSlotBytes + kBatch * 4 + 16 * lane);
      } else {
        load_batch_in(cur, rw, mk, (int64_t)t0 + kTokLane * lane, lo, hi, vec);
      }
      c_slot = c_slot + 1 == kUSlots ? 0 : c_slot + 1;
      ++c_n;
      // every lane has read the slot consumed before this one: lane 0 refills it
      __syncwarp();
      if (lane == 0) produce(kc, c_n);
      // the next unit's window, once it is queued (its loads complete behind this unit)
      if (!nx_loaded) {
        const int nc = __shfl_sync(kFull, p_nclaim, 0);
        if (nc > kc + 1) {
          __syncwarp();
          const UnitQ nu = q[(kc + 1) & (kUQ - 1)];
          if (nu.ri >= 0) nws = load_window(nu, nu.p1);
          nx_loaded = true;
        }
      }
      const uint32_t mk16 = nonzero_bytes4(cur.m.x) | nonzero_bytes4(cur.m.y) << 4 |
                            nonzero_bytes4(cur.m.z) << 8 | nonzero_bytes4(cur.m.w) << 12;
      const bool whole = tb >= 0 && tb + kBatch <= ulen;
      float out[kTokLane];  // physical order when fast, else logical
      uint32_t on16, st16 = 0xffffu;  // tokens counted / stored (same order as out)
      bool phys;
      if (__all_sync(kFull, e == 0u) && whole) {
        // constant slopes: no sequence end, every token inside the unit.  Chunk k's map is
        // x -> S_k + gamma^4 x; the lane map composes the chunks in logical order.
        phys = true;
        on16 = ((mk16 | mk16 << 16) >> (4 * prot)) & 0xffffu;  // physical mask nibbles
        float v[kTokLane];
#pragma unroll
        for (int i = 0; i < kTokLane; ++i) v[i] = (on16 >> i) & 1u ? tok_r(cur, i) : 0.f;
        float Sk[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
          Sk[k] = fmaf(gamma, fmaf(gamma, fmaf(gamma, v[4 * k + 3], v[4 * k + 2]), v[4 * k + 1]), v[4 * k]);
        float u[4], L[4];  // L[c] = Sk[(c - prot) & 3]
#pragma unroll
        for (int c = 0; c < 4; ++c) u[c] = (prot & 1) ? Sk[(c + 3) & 3] : Sk[c];
#pragma unroll
        for (int c = 0; c < 4; ++c) L[c] = (prot & 2) ? u[(c + 2) & 3] : u[c];
        const float S = fmaf(a.g4, fmaf(a.g4, fmaf(a.g4, L[3], L[2]), L[1]), L[0]);
        float sS = S;
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const float o = __shfl_down_sync(kFull, sS, 1 << k);
          if (lane + (1 << k) < 32) sS = fmaf(a.gpw[k], o, sS);
        }
        float rS = __shfl_down_sync(kFull, sS, 1);
        if (lane == 31) rS = 0.f;
        const float tS = __shfl_sync(kFull, sS, 0);
        float C[4];  // G right of logical chunk c
        C[3] = fmaf(rPl, carry, rS);
        C[2] = fmaf(a.g4, C[3], L[3]);
        C[1] = fmaf(a.g4, C[2], L[2]);
        C[0] = fmaf(a.g4, C[1], L[1]);
        float D[4];  // D[k] = C[(k + prot) & 3]
#pragma unroll
        for (int k = 0; k < 4; ++k) u[k] = (prot & 1) ? C[(k + 1) & 3] : C[k];
#pragma unroll
        for (int k = 0; k < 4; ++k) D[k] = (prot & 2) ? u[(k + 2) & 3] : u[k];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          out[4 * k + 3] = fmaf(gamma, D[k], v[4 * k + 3]);
          out[4 * k + 2] = fmaf(gamma, out[4 * k + 3], v[4 * k + 2]);
          out[4 * k + 1] = fmaf(gamma, out[4 * k + 2], v[4 * k + 1]);
          out[4 * k] = fmaf(gamma, out[4 * k + 1], v[4 * k]);
        }
        carry = fmaf(a.g512, carry, tS);
      } else {
        // general: sequence ends (slope 0 at a sequence's last token) and the unit's bounds,
        // token by token in logical order
        phys = false;
        {
          float4 u4[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) u4[c] = (prot & 1) ? cur.r[(c + 3) & 3] : cur.r[c];
#pragma unroll
          for (int c = 0; c < 4; ++c) cur.r[c] = (prot & 2) ? u4[(c + 2) & 3] : u4[c];
        }
        uint32_t in16 = 0xffffu;
        if (lt < 0) in16 &= lt + kTokLane <= 0 ? 0u : (0xffffu << (uint32_t)(-lt)) & 0xffffu;
        if (lt + kTokLane > ulen) in16 &= lt >= ulen ? 0u : 0xffffu >> (uint32_t)(lt + kTokLane - ulen);
        on16 = in16 & mk16;
        float v[kTokLane];
#pragma unroll
        for (int i = 0; i < kTokLane; ++i) v[i] = (on16 >> i) & 1u ? tok_r(cur, i) : 0.f;
        float S = 0.f;
#pragma unroll
        for (int i = kTokLane - 1; i >= 0; --i) S = fmaf(((e >> i) & 1u) ? 0.f : gamma, S, v[i]);
        float rS, rP, bS, bP;
        warp_compose(S, e ? 0.f : a.gpw[0], lane, rS, rP, bS, bP);
        float g_next = rS + rP * carry;
#pragma unroll
        for (int i = kTokLane - 1; i >= 0; --i) {
          out[i] = fmaf(((e >> i) & 1u) ? 0.f : gamma, g_next, v[i]);
          g_next = out[i];
        }
        carry = bS + bP * carry;
        st16 = in16;
      }
      if (count_stats) {
        float sa = 0.f, sb = 0.f, qa = 0.f, qb = 0.f;
#pragma unroll
        for (int i = 0; i < kTokLane; i += 2) {
          const float o0 = (on16 >> i) & 1u ? out[i] : 0.f;
          const float o1 = (on16 >> (i + 1)) & 1u ? out[i + 1] : 0.f;
          sa += o0;
          qa = fmaf(o0, o0, qa);
          sb += o1;
          qb = fmaf(o1, o1, qb);
        }
        s_m += (double)__popc(on16);
        s_g += (double)(sa + sb);
        s_g2 += (double)(qa + qb);
      }
      const int srot = phys ? prot : 0;  // out chunk k holds logical chunk (k + srot) & 3
      if (vstore && st16 == 0xffffu) {
        float4* gp = reinterpret_cast<float4*>(G + lt);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          __stcs(gp + ((k + srot) & 3), make_float4(out[4 * k], out[4 * k + 1], out[4 * k + 2], out[4 * k + 3]));
      } else {
        float* gp = G + lt;
#pragma unroll
        for (int i = 0; i < kTokLane; ++i)
          if ((st16 >> i) & 1u) gp[4 * (((i >> 2) + srot) & 3) + (i & 3)] = out[i];
      }
    }
    // per-sequence returns G_0 of the unit's sequences [p0, p1)
    float* SR = a.seq_return[r];
    if (SR != nullptr) {
      __syncwarp();  // this warp's G stores precede the reads
      const int64_t gs = rt.gs[ri];
      if (wtop == cu.p1 && cu.p1 - cu.p0 <= 32) {
        // the window still holds every start: lane j takes sequence p1 - 1 - j
        const int p = cu.p1 - 1 - lane;
        const int s_next = ws;                                  // start of p + 1
        int s = __shfl_down_sync(kFull, ws, 1);                 // start of p
        if (p == cu.p0) s = 0;
        if (p >= cu.p0) SR[p - gs] = s_next > s ? G[s] : 0.f;
      } else {
        unit_seq_returns(SR, G - ua, cum, cum[gs], gs, cu.p0, cu.p1, lane);
      }
    }
    // the next unit
    if (lane == 0) {
      while (p_nclaim <= kc + 1 && !p_done) claim();
    }
    __syncwarp();
    cu = q[(kc + 1) & (kUQ - 1)];
    if (cu.ri >= 0) ws = nx_loaded ? nws : load_window(cu, cu.p1);
    nx_loaded = false;
    // keep kUSlots - 1 batches in flight
    if (lane == 0) produce(kc + 1, c_n);
    __syncwarp();
  }
  returns_epilogue(a, rt, red, s_m, s_g, s_g2, kWarps);
}

// ---------------------------------------------------------------------------------------
// returns_coop_kernel: small and mid batches (C2, C4), where the look-back chains of the
// windowed kernel are latency-bound.  A co-resident grid gives every window of 512 * nb tokens
// (nb = 1, 2 or 4: the smallest that fits) its own warp.  The warp loads its window into shared
// memory once (TMA bulk copies; the buffer's last few tokens by lanes), composes the window's map
// (pass 1) and publishes it; after one grid barrier every window's map is final, so the carry into
// a window is the composition of the maps to its right up to the first zero slope (a sequence end
// or the rank's end), read 32 windows per round trip with no waiting; pass 2 turns the lane maps
// into the returns from the same shared-memory copy.  Each token is read from HBM once and written
// once.  Chosen by choose_returns when the windows fit the grid.
// ---------------------------------------------------------------------------------------

constexpr int kCWinMax = kBatch * kCoopMaxNB;       // 2048 tokens
constexpr int kCBytes = kCWinMax * 4 + kCWinMax;    // a window's rewards, then its mask bytes
#ifndef EARL_AGG_CCTAS
#define EARL_AGG_CCTAS 2
#endif
constexpr int kCCtas = EARL_AGG_CCTAS;

__global__ void __launch_bounds__(kWarps * 32, kCCtas) returns_coop_kernel(const __grid_constant__ AggArgs a) {
  __shared__ RankTable rt;
  __shared__ uint32_t ends_bm[kWarps][kCWinMax / 32];
  __shared__ float2 lmap[kWarps][kCoopMaxNB][32];  // per batch and lane: exclusive suffix map
  __shared__ float2 bmap[kWarps][kCoopMaxNB];      // per batch: its map
  __shared__ double red[3][32];
  __shared__ uint64_t cbar[kWarps];
  __shared__ int s_ok;
  extern __shared__ __align__(128) uint8_t cmem[];  // [kWarps][kCBytes]
  if (gated_out(a)) return;
  if (threadIdx.x < 32) {
    int nb = a.coop_nb;
    if (nb <= 0) device_choice(a, &nb);
    rank_table(a, rt, 1, nb > 0 ? nb : kCoopMaxNB);
    const int64_t total = rt.wbeg[rt.n];
    const bool ok = nb > 0 && total <= (int64_t)gridDim.x * kWarps && total <= a.win_cap;
    if (threadIdx.x == 0) s_ok = ok;
    if (!ok && threadIdx.x == 0 && blockIdx.x == 0)
      latch(a.plan.hdr, EARL_ERR_CAPACITY, (int)min(total, (int64_t)INT32_MAX));
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int64_t total = s_ok ? rt.wbeg[rt.n] : 0;
  const int64_t win = (int64_t)kBatch * rt.nb;
  const float gamma = a.gamma;
  const float g16 = a.gamma16;
  float2* agg = reinterpret_cast<float2*>(a.win);  // the window maps (no tags: a barrier orders them)
  uint32_t* bm = ends_bm[wid];
  uint8_t* buf = cmem + (size_t)wid * kCBytes;
  const uint32_t bar = smem_addr(&cbar[wid]);
  double s_m = 0.0, s_g = 0.0, s_g2 = 0.0;

  const int64_t gw = (int64_t)blockIdx.x * kWarps + wid;  // this warp's window
  const bool has = gw < total;
  int ri = 0;
  if (has) while (gw >= rt.wbeg[ri + 1]) ++ri;
  const int r = has ? rt.rank[ri] : 0;
  const int64_t ntok = has ? rt.ntok[ri] : 0;
  const int64_t w0 = has ? (gw - rt.wbeg[ri]) * win : 0;
  const int64_t w1 = has ? min(ntok, w0 + win) : 0;
  const int n = (int)(w1 - w0);                     // tokens of the window
  const int nb = (n + kBatch - 1) / kBatch;
  const float* rw = has ? a.rewards[r] : nullptr;
  const uint8_t* mk = has ? a.mask[r] : nullptr;
  float* G = has ? a.returns[r] : nullptr;
  const int64_t* cum = a.plan.cum[0];
  const int64_t gs = has ? rt.gs[ri] : 0, pend = has ? gs + rt.cnt[ri] : 0;
  const int64_t base = has ? cum[gs] : 0;

  // ---- the window into shared memory: rewards [0, 4n) B, mask [4 * kCWinMax, + n) B -------
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const bool vec = has && aligned(rw, 16) && aligned(mk, 16);
  const int nr = vec ? (n & ~3) : 0, nm = vec ? (n & ~15) : 0;  // by TMA (whole 16-B granules)
  if (lane == 0) {
    if (nr + nm > 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                   "r"((uint32_t)(nr * 4 + nm)) : "memory");
      if (nr > 0)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(smem_addr(buf)), "l"(rw + w0), "r"((uint32_t)(nr * 4)), "r"(bar) : "memory");
      if (nm > 0)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(smem_addr(buf + kCWinMax * 4)), "l"(mk + w0), "r"((uint32_t)nm), "r"(bar) : "memory");
    } else {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
    }
  }
  float* sr = reinterpret_cast<float*>(buf);
  uint8_t* sm = buf + kCWinMax * 4;
  for (int t = nr + lane; t < n; t += 32) sr[t] = rw[w0 + t];
  for (int t = nm + lane; t < n; t += 32) sm[t] = mk[w0 + t];
  // sequence ends inside the window (token s - 1 for every start s in (w0, w1]) while the copy lands
  const int64_t lo = has ? mark_ends(bm, nb * (kBatch / 32), cum, base, gs, pend, w0, w1, lane) : 0;
  {
    uint32_t done;
    do {
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
          " selp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done) : "r"(bar), "r"(0u) : "memory");
    } while (!done);
  }
  __syncwarp();

  // batch b of the window from shared memory (rotated chunk order: conflict-free), tokens past
  // the window's end masked off
  const int rot = (lane >> 1) & 3;
  auto get = [&](Batch& B, int b, uint32_t& on16) {
    const uint8_t* rb = buf + b * (kBatch * 4) + 64 * lane;
    float4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = *reinterpret_cast<const float4*>(rb + 16 * ((k + rot) & 3));
    float4 u[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) u[c] = (rot & 1) ? v[(c + 3) & 3] : v[c];
#pragma unroll
    for (int c = 0; c < 4; ++c) B.r[c] = (rot & 2) ? u[(c + 2) & 3] : u[c];
    B.m = *reinterpret_cast<const uint4*>(sm + b * kBatch + 16 * lane);
    const int lt = b * kBatch + kTokLane * lane;
    uint32_t in16 = 0xffffu;
    if (lt + kTokLane > n) in16 = lt >= n ? 0u : 0xffffu >> (uint32_t)(lt + kTokLane - n);
    on16 = in16 & (nonzero_bytes4(B.m.x) | nonzero_bytes4(B.m.y) << 4 | nonzero_bytes4(B.m.z) << 8 |
                   nonzero_bytes4(B.m.w) << 12);
  };
  auto ends16 = [&](int b) { return (bm[16 * b + (lane >> 1)] >> (16 * (lane & 1))) & 0xffffu; };

  // ---- pass 1: lane maps, batch maps, the window's map -------------------------------------
  float wS = 0.f, wP = 1.f;
#pragma unroll 1
  for (int b = nb - 1; b >= 0; --b) {
    Batch cur;
    uint32_t on16;
    get(cur, b, on16);
    const uint32_t e = ends16(b);
    float S = 0.f;
#pragma unroll
    for (int i = kTokLane - 1; i >= 0; --i)
      S = fmaf(((e >> i) & 1u) ? 0.f : gamma, S, (on16 >> i) & 1u ? tok_r(cur, i) : 0.f);
    float rS, rP, bS, bP;
    warp_compose(S, e ? 0.f : g16, lane, rS, rP, bS, bP);
    lmap[wid][b][lane] = make_float2(rS, rP);
    if (lane == 0) bmap[wid][b] = make_float2(bS, bP);
    wS = bS + bP * wS;
    wP = bP * wP;
  }
  if (has && lane == 0) agg[gw] = make_float2(wS, wP);
  delay_inject(9);
  // every window's map is published
  if (gridDim.x == 1) __syncthreads();
  else cooperative_groups::this_grid().sync();

  if (has) {
    // ---- carry: the maps of the windows to the right (same rank) up to the first zero slope
    const int64_t wend = rt.wbeg[ri + 1];
    float cS = 0.f, cP = 1.f;
    for (int64_t j0 = gw + 1; j0 < wend && cP != 0.f; j0 += 32) {
      const int64_t j = j0 + lane;
      const float2 m = j < wend ? __ldcg(&agg[j]) : make_float2(0.f, 1.f);
      float rS, rP, tS, tP;
      warp_compose(m.x, m.y, lane, rS, rP, tS, tP);
      cS = cS + cP * tS;
      cP = cP * tP;
    }
    // ---- pass 2: the returns, float4 stores, statistics
    const bool count_stats = rt.t[ri] == 0;
    float c = cS;  // G right of batch b (right to left)
#pragma unroll 1
    for (int b = nb - 1; b >= 0; --b) {
      Batch cur;
      uint32_t on16;
      get(cur, b, on16);
      const uint32_t e = ends16(b);
      const float2 rm = lmap[wid][b][lane];
      float g_next = rm.x + rm.y * c;
      float out[kTokLane];
#pragma unroll
      for (int i = kTokLane - 1; i >= 0; --i) {
        out[i] = fmaf(((e >> i) & 1u) ? 0.f : gamma, g_next, (on16 >> i) & 1u ? tok_r(cur, i) : 0.f);
        g_next = out[i];
      }
      const float2 bmb = bmap[wid][b];
      c = bmb.x + bmb.y * c;
      if (count_stats) {
        float sa = 0.f, sb = 0.f, qa = 0.f, qb = 0.f;
#pragma unroll
        for (int i = 0; i < kTokLane; i += 2) {
          const float o0 = (on16 >> i) & 1u ? out[i] : 0.f;
          const float o1 = (on16 >> (i + 1)) & 1u ? out[i + 1] : 0.f;
          sa += o0;
          qa = fmaf(o0, o0, qa);
          sb += o1;
          qb = fmaf(o1, o1, qb);
        }
        s_m += (double)__popc(on16);
        s_g += (double)(sa + sb);
        s_g2 += (double)(qa + qb);
      }
      const int64_t t = w0 + b * kBatch + kTokLane * lane;
      if (aligned(G, 16) && t + kTokLane <= w1) {
        float4* gp = reinterpret_cast<float4*>(G + t);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          __stcs(gp + k, make_float4(out[4 * k], out[4 * k + 1], out[4 * k + 2], out[4 * k + 3]));
      } else {
        for (int i = 0; i < kTokLane; ++i)
          if (t + i < w1) G[t + i] = out[i];
      }
    }
    // per-sequence return G_0 of the sequences starting in the window
    seq_returns(a.seq_return[r], G, cum, base, gs, pend, lo, w1, ntok, lane);
    __syncwarp();
  }
  returns_epilogue(a, rt, red, s_m, s_g, s_g2, kWarps);
}

// A_t = m_t (G_t - mu) / (sigma + eps) over every token of the launch's source ranks: one
// flattened stream of 4-token quads over all ranks (4 quads in flight per thread), then the
// unaligned remainders token by token.  Measured on the C5-lt batch: read-only-path loads
// (ld.global.nc) and a grid sized to the work (launch_advantages) 0.50 ms, against 0.58 ms with
// evict-first loads and 8 CTAs per SM.
__global__ void __launch_bounds__(256) advantage_kernel(const __grid_constant__ AggArgs a) {
  __shared__ RankTable rt;
  __shared__ int64_t qbeg[kMaxWorld + 1];   // vector quads of the ranks (prefix)
  __shared__ int64_t tbeg[kMaxWorld + 1];   // scalar remainder tokens of the ranks (prefix)
  __shared__ float s_mu, s_inv;
  if (threadIdx.x < 32) {
    // the statistics are loaded first, so their round trip overlaps the header's
    double st[3] = {0.0, 0.0, 0.0};
    if (threadIdx.x == 0) { st[0] = a.stats[0]; st[1] = a.stats[1]; st[2] = a.stats[2]; }
    rank_table(a, rt, 1);
    if (threadIdx.x == 0) {
    qbeg[0] = tbeg[0] = 0;
    for (int ri = 0; ri < rt.n; ++ri) {
      const int r = rt.rank[ri];
      const bool vec = aligned(a.returns[r], 16) && aligned(a.adv[r], 16) && aligned(a.mask[r], 4);
      const int64_t nq = vec ? rt.ntok[ri] >> 2 : 0;
      qbeg[ri + 1] = qbeg[ri] + nq;
      tbeg[ri + 1] = tbeg[ri] + rt.ntok[ri] - 4 * nq;
    }
    const double n = st[0];
    const double mu = n > 0 ? st[1] / n : 0.0;
    double var = n > 0 ? st[2] / n - mu * mu : 0.0;
    if (var < 0) var = 0;
    s_mu = (float)mu;
    s_inv = (float)(1.0 / (sqrt(var) + (double)a.eps));
    }
  }
  __syncthreads();
  const float mu = s_mu, inv = s_inv;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t Q = qbeg[rt.n];
  constexpr int kU = 4;
  int ri = 0;  // rank cursor: q only grows
  for (int64_t q0 = tid; q0 < Q; q0 += kU * stride) {
    float4 g[kU];
    uint32_t m[kU];
    int rr[kU];
    int64_t qq[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t q = q0 + u * stride;
      rr[u] = -1;
      if (q < Q) {
        while (q >= qbeg[ri + 1]) ++ri;
        rr[u] = rt.rank[ri];
        qq[u] = q - qbeg[ri];
        g[u] = __ldg(reinterpret_cast<const float4*>(a.returns[rr[u]]) + qq[u]);
        m[u] = __ldg(reinterpret_cast<const unsigned int*>(a.mask[rr[u]]) + qq[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (rr[u] < 0) continue;
      float4 o;
      o.x = (m[u] & 0xffu) ? (g[u].x - mu) * inv : 0.f;
      o.y = (m[u] & 0xff00u) ? (g[u].y - mu) * inv : 0.f;
      o.z = (m[u] & 0xff0000u) ? (g[u].z - mu) * inv : 0.f;
      o.w = (m[u] & 0xff000000u) ? (g[u].w - mu) * inv : 0.f;
      __stcs(reinterpret_cast<float4*>(a.adv[rr[u]]) + qq[u], o);
    }
  }
  const int64_t Tt = tbeg[rt.n];
  for (int64_t j = tid; j < Tt; j += stride) {
    int ri = 0;
    while (j >= tbeg[ri + 1]) ++ri;
    const int r = rt.rank[ri];
    const int64_t t = rt.ntok[ri] - (tbeg[ri + 1] - j);  // the remainder is the rank's tail
    a.adv[r][t] = a.mask[r][t] ? (a.returns[r][t] - mu) * inv : 0.f;
  }
}

}  // namespace

int64_t returns_windows(int64_t tokens) { return (tokens + kMaxWin - 1) / kMaxWin + 16384; }

cudaError_t launch_returns_units(const AggArgs& a, int sm_count, cudaStream_t s) {
  unit_table_kernel<<<sm_count * 4, 256, 0, s>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  constexpr size_t kRingBytes = (size_t)kWarps * kUSlots * kSlotBytes;
  static bool opted[64] = {};
  e = opt_in_dynamic_smem(returns_units_kernel, (int)kRingBytes, opted);
  if (e != cudaSuccess) return e;
  returns_units_kernel<<<sm_count * kU2Ctas, kWarps * 32, kRingBytes, s>>>(a);
  return cudaGetLastError();
}

int returns_coop_capacity_warps(int sm_count) {
  static int per_sm[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  const int d = dev >= 0 && dev < 64 ? dev : 0;
  if (per_sm[d] <= 0) {
    static bool opted[64] = {};
    if (opt_in_dynamic_smem(returns_coop_kernel, (int)(kWarps * kCBytes), opted) != cudaSuccess) {
      (void)cudaGetLastError();
      return 0;
    }
    int p = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p, returns_coop_kernel, kWarps * 32,
                                                      kWarps * kCBytes) != cudaSuccess)
      p = 0;
    (void)cudaGetLastError();
    per_sm[d] = p > kCCtas ? kCCtas : p;
    if (per_sm[d] <= 0) return 0;
  }
  return sm_count * per_sm[d] * kWarps;
}

// One warp per window: ceil(windows / 8) CTAs (windows <= 0: the whole co-resident grid, for a
// launch that decides on the device).
cudaError_t launch_returns_coop(const AggArgs& a, int64_t windows, int sm_count, cudaStream_t s) {
  static bool opted[64] = {};
  cudaError_t e = opt_in_dynamic_smem(returns_coop_kernel, (int)(kWarps * kCBytes), opted);
  if (e != cudaSuccess) return e;
  const int64_t cap = returns_coop_capacity_warps(sm_count) / kWarps;
  int64_t g = windows > 0 ? (windows + kWarps - 1) / kWarps : cap;
  if (g > cap) g = cap;
  const int grid = (int)(g < 1 ? 1 : g);
  if (grid <= 1) {
    returns_coop_kernel<<<1, kWarps * 32, kWarps * kCBytes, s>>>(a);
    return cudaGetLastError();
  }
  void* args[] = {const_cast<AggArgs*>(&a)};
  return cudaLaunchCooperativeKernel((const void*)returns_coop_kernel, dim3(grid), dim3(kWarps * 32),
                                     args, kWarps * kCBytes, s);
}

cudaError_t launch_returns(const AggArgs& a, int sm_count, cudaStream_t s) {
  // the batch ring: kSlots x 2.5 KB per warp of dynamic shared memory; with the static arrays
  // it exceeds the 48 KB a launch gets without opting in
  constexpr size_t kRingBytes = EARL_AGG_TMA ? (size_t)kWarps * kSlots * kSlotBytes : 0;
  if (kRingBytes > 0) {
    static bool opted[64] = {};
    cudaError_t e = opt_in_dynamic_smem(returns_kernel, (int)kRingBytes, opted);
    if (e != cudaSuccess) return e;
  }
  returns_kernel<<<sm_count * kCtasPerSm, kWarps * 32, kRingBytes, s>>>(a);
  return cudaGetLastError();
}

// Grid sized to the work when the plan's token count is known on the host (tokens >= 0): about
// EARL_ADV_TRIPS loop trips of kU quads per thread, at least one CTA per SM and at most 64 per SM
// (C5-lt: 0.50 ms at 64 per SM against 0.52 at 16).  2 trips since the rank table costs one
// round trip per CTA (C2 / C4 12.3 -> 10.2 / 14.3 -> 12.3 us against 8 trips; 1 or 4: no better).
#ifndef EARL_ADV_TRIPS
#define EARL_ADV_TRIPS 2
#endif
cudaError_t launch_advantages(const AggArgs& a, int sm_count, int64_t tokens, cudaStream_t s) {
  int64_t grid = (int64_t)sm_count * 16;
  if (tokens >= 0) {
    grid = (tokens / 4 + 256 * 4 * EARL_ADV_TRIPS - 1) / (256 * 4 * EARL_ADV_TRIPS);
    grid = grid < sm_count ? sm_count : (grid > 64LL * sm_count ? 64LL * sm_count : grid);
  }
  advantage_kernel<<<(unsigned)grid, 256, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace earl
