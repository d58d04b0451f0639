// planner.cu -- device-side dispatch planner.
//
// One cooperative grid of G CTAs x 1024 threads computes the whole plan in phases separated by
// grid-wide barriers.  G scales with the batch (G = ceil(N / 4096), at most one CTA per SM), so
// the configs' N <= 512 run as a single CTA (barriers degenerate to __syncthreads) while the
// bandwidth sweep's 4e5 sequences spread over ~100 SMs.  There is no host synchronisation, and
// the plan is bit-for-bit deterministic for any G (integer arithmetic only; every scan and
// partition is order-defined), so every rank computes the identical plan from identical lengths.
//
// Phases ("adaptive to the current data distribution layout and parallelism
// configuration"; the steps follow SURVEY.md §8(c) and the readings in DESIGN.md §2):
//   0  P = exclusive scan of L (int64), T = sum L; latch L_i < 0 (reading c20)
//   1  g(i) for src and dst: GIVEN_COUNTS / CONTIG midpoint / LPT / EXPLICIT (reading c4)
//   2  per layout: stable partition of sequences by group (ascending i inside a group, c5);
//      per SP chunk k: scan of BLOCK chunk lengths in that order -> local token offsets (c7)
//   3  pieces: two-pointer intersection of the src and dst chunk partitions of every sequence
//   4  stable partition of pieces by message key (src shard, dst shard); message token offsets
//   5  per-(rank, shard) record / token bases, message byte offsets (16-B aligned field blocks)
//   6  records: piece x sending replica ts < min(TP_src, TP_dst) (reading c9), in (s, ds, i, x)
//
// Grid-wide primitives: grid_scan (per-CTA reduce -> barrier -> per-CTA carry from the CTA
// sums -> block scans with carry) and grid_partition (per-CTA key histograms -> barrier ->
// per-(key, CTA) bases -> stable in-CTA ranks via __match_any_sync).
#include <cooperative_groups.h>

#include "earl_internal.cuh"

namespace cg = cooperative_groups;

namespace earl {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int NT = kPlanThreads;
constexpr int kItems = 4;

__device__ __forceinline__ void latch(PlanHeader* h, int code, int detail) {
  if (atomicCAS(&h->err, 0, code) == 0) h->err_detail = detail;
}

__device__ __forceinline__ void stamp(const PlanArgs& a, int k) {
  if (a.phase_ts != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.phase_ts[k] = t;
  }
}

// The CTA's largest length into h->max_len (values >= 0).
__device__ __forceinline__ void publish_max_len(PlanHeader* h, uint32_t m, unsigned* s_max) {
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0) atomicMax(s_max, m);
  __syncthreads();
  if (threadIdx.x == 0 && *s_max) atomicMax(reinterpret_cast<unsigned long long*>(&h->max_len),
                                            (unsigned long long)*s_max);
}

__device__ __forceinline__ void gsync() {
  delay_inject(6);
  if (gridDim.x == 1) __syncthreads();
  else cg::this_grid().sync();
}

__device__ __forceinline__ int64_t range_lo(int64_t n) { return n * blockIdx.x / gridDim.x; }
__device__ __forceinline__ int64_t range_hi(int64_t n) { return n * (blockIdx.x + 1) / gridDim.x; }

// BLOCK rule: q = L / sp, r = L % sp, chunk k = [k*q + min(k,r), (k+1)*q + min(k+1,r)).
// Sequence lengths are int32 (the C ABI's seq_lens), so the division is 32-bit.
__device__ __forceinline__ int64_t chunk_lo(int64_t L, int sp, int k) {
  const uint32_t q = (uint32_t)L / (uint32_t)sp, r = (uint32_t)L - q * (uint32_t)sp;
  return (int64_t)k * q + ((uint32_t)k < r ? (uint32_t)k : r);
}
__device__ __forceinline__ int64_t chunk_len(int64_t L, int sp, int k) {
  const uint32_t q = (uint32_t)L / (uint32_t)sp, r = (uint32_t)L - q * (uint32_t)sp;
  return (int64_t)q + ((uint32_t)k < r ? 1 : 0);
}

// Block-wide exclusive scan of one int64 per thread.  sm: [NT/32 + 1].
__device__ int64_t block_excl_scan(int64_t v, int64_t& total, int64_t* sm) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sm[w] = x;
  __syncthreads();
  if (w == 0) {
    const int64_t s = (lane < NT / 32) ? sm[lane] : 0;
    int64_t inc = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(kFull, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane < NT / 32) sm[lane] = inc - s;
    if (lane == 31) sm[NT / 32] = inc;
  }
  __syncthreads();
  const int64_t res = sm[w] + x - v;
  total = sm[NT / 32];
  __syncthreads();
  return res;
}

// Exclusive scan over [lo, hi) starting from `carry`: put(i, carry + sum_{lo<=j<i} get(j)).
// Returns the range's sum.
template <class Get, class Put>
__device__ int64_t tile_scan_range(int64_t lo, int64_t hi, int64_t carry, Get get, Put put,
                                   int64_t* sm) {
  int64_t sum = 0;
  for (int64_t base = lo; base < hi; base += (int64_t)NT * kItems) {
    int64_t v[kItems];
    int64_t tsum = 0;
    const int64_t i0 = base + (int64_t)threadIdx.x * kItems;
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      v[it] = (i0 + it < hi) ? get(i0 + it) : 0;
      tsum += v[it];
    }
    int64_t total;
    int64_t run = carry + sum + block_excl_scan(tsum, total, sm);
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      if (i0 + it < hi) put(i0 + it, run);
      run += v[it];
    }
    sum += total;
  }
  return sum;
}

// Grid-wide exclusive scan over [0, n).  `get` must be pure (it runs twice when G > 1) and
// read only data published before the call; outputs of `put` are visible to other CTAs after
// the caller's next gsync().  Returns the total (in every CTA).
template <class Get, class Put>
__device__ int64_t grid_scan(int64_t n, Get get, Put put, int64_t* cta_sums, int64_t* sm) {
  const int64_t lo = range_lo(n), hi = range_hi(n);
  if (gridDim.x == 1) return tile_scan_range(lo, hi, 0, get, put, sm);
  int64_t part = 0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += NT) part += get(i);
  int64_t total;
  block_excl_scan(part, total, sm);
  if (threadIdx.x == 0) cta_sums[blockIdx.x] = total;
  gsync();
  // carry = sum of the CTAs before this one; grand total (warp 0)
  __shared__ int64_t s_carry, s_total;
  if (threadIdx.x < 32) {
    int64_t before = 0, all = 0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) {
      const int64_t v = cta_sums[b];
      all += v;
      if (b < (int)blockIdx.x) before += v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      before += __shfl_xor_sync(kFull, before, o);
      all += __shfl_xor_sync(kFull, all, o);
    }
    if (threadIdx.x == 0) { s_carry = before; s_total = all; }
  }
  __syncthreads();
  const int64_t carry = s_carry, grand = s_total;
  tile_scan_range(lo, hi, carry, get, put, sm);
  return grand;
}

struct PartitionSmem {
  int32_t whist[NT / 32][kMaxKeys];
  int64_t running[kMaxKeys];
  int64_t tile_tot[kMaxKeys];
  int64_t bstart[kMaxKeys + 1];
  int64_t before[kMaxKeys];
  int64_t tot[kMaxKeys];
  unsigned hist[kMaxKeys];
};

// Grid-wide stable counting sort of [0, n) by key(i) in [0, K), K <= 64: emit(i, position).
// On return ps.bstart[0..K] holds the global bucket starts (same in every CTA).  Positions are
// visible to other CTAs after the caller's next gsync().
template <class KeyF, class Emit>
__device__ void grid_partition(int64_t n, int K, KeyF key, Emit emit, int32_t* ghist,
                               PartitionSmem& ps) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t lo = range_lo(n), hi = range_hi(n);
  if (tid < kMaxKeys) ps.hist[tid] = 0;
  __syncthreads();
  for (int64_t i = lo + tid; i < hi; i += NT) atomicAdd(&ps.hist[key(i)], 1u);
  __syncthreads();
  if (gridDim.x == 1) {
    if (tid < K) { ps.tot[tid] = ps.hist[tid]; ps.before[tid] = 0; }
  } else {
    if (tid < K) ghist[(int64_t)blockIdx.x * kMaxKeys + tid] = (int32_t)ps.hist[tid];
    gsync();
    if (tid < K) {
      int64_t before = 0, all = 0;
      for (int b = 0; b < (int)gridDim.x; ++b) {
        const int64_t v = ghist[(int64_t)b * kMaxKeys + tid];
        all += v;
        if (b < (int)blockIdx.x) before += v;
      }
      ps.tot[tid] = all;
      ps.before[tid] = before;
    }
  }
  __syncthreads();
  if (tid == 0) {
    int64_t acc = 0;
    for (int k = 0; k < K; ++k) { ps.bstart[k] = acc; acc += ps.tot[k]; }
    ps.bstart[K] = acc;
  }
  if (tid < K) ps.running[tid] = ps.before[tid];
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t base = lo; base < hi; base += NT) {
    const int64_t i = base + tid;
    const int k = (i < hi) ? key(i) : -1;
    ps.whist[w][lane] = 0;
    ps.whist[w][lane + 32] = 0;
    __syncwarp();
    const unsigned peers = __match_any_sync(kFull, k);
    const int rank = __popc(peers & lt);
    if (k >= 0 && rank == 0) ps.whist[w][k] = __popc(peers);
    __syncthreads();
    if (tid < K) {
      int32_t acc = 0;
      for (int ww = 0; ww < NT / 32; ++ww) {
        const int32_t c = ps.whist[ww][tid];
        ps.whist[ww][tid] = acc;
        acc += c;
      }
      ps.tile_tot[tid] = acc;
    }
    __syncthreads();
    if (k >= 0) emit(i, ps.bstart[k] + ps.running[k] + ps.whist[w][k] + rank);
    __syncthreads();
    if (tid < K) ps.running[tid] += ps.tile_tot[tid];
    __syncthreads();
  }
}

// The planner's code runs once per plan in a single CTA for the configs' N, so its latency is
// dominated by instruction fetch: every scan and partition therefore goes through ONE
// non-inlined copy of these two routines over plain arrays (values / keys precomputed by
// small elementwise passes), instead of one inlined instantiation per call site.
__device__ __noinline__ int64_t scan_array(const int64_t* vals, int64_t* out, int64_t n,
                                           int64_t* cta_sums, int64_t* sm) {
  return grid_scan(
      n, [&](int64_t i) { return vals[i]; }, [&](int64_t i, int64_t ex) { out[i] = ex; }, cta_sums,
      sm);
}

__device__ __noinline__ void partition_array(const int32_t* keys, int64_t n, int K,
                                             int32_t* perm_out, int32_t* ghist,
                                             PartitionSmem& ps) {
  grid_partition(
      n, K, [&](int64_t i) { return keys[i]; },
      [&](int64_t i, int64_t pos) { perm_out[pos] = (int32_t)i; }, ghist, ps);
}

// 64-bit BLOCK split (FLAT splits a whole group's token stream, which may exceed 2^32).
__device__ __forceinline__ int64_t block_lo64(int64_t S, int sp, int k) {
  const int64_t q = S / sp, r = S - q * sp;
  return (int64_t)k * q + ((int64_t)k < r ? (int64_t)k : r);
}

// The virtual chunks of one sequence under one layout's SP split (readings c7, n1-n3).  They are
// consecutive intervals covering [0, L) in chunk order; chunk c is held by SP rank owner(c).
struct Chunker {
  int split, sp, C;      // C virtual chunks: 2*sp for ZIGZAG, sp otherwise
  int64_t L;
  int64_t gpos, S;       // FLAT: the sequence's offset in its group stream, the stream length
  int owner_short;       // THRESHOLD: the SP rank holding a short sequence whole, else -1

  __device__ __forceinline__ int owner(int c) const {
    return (split == EARL_SP_ZIGZAG && c >= sp) ? 2 * sp - 1 - c : c;
  }
  __device__ __forceinline__ void bounds(int c, int64_t& lo, int64_t& hi) const {
    if (split == EARL_SP_ZIGZAG) {
      lo = chunk_lo(L, 2 * sp, c);
      hi = lo + chunk_len(L, 2 * sp, c);
    } else if (split == EARL_SP_FLAT) {
      const int64_t a = block_lo64(S, sp, c) - gpos, b = block_lo64(S, sp, c + 1) - gpos;
      lo = a < 0 ? 0 : (a > L ? L : a);
      hi = b < 0 ? 0 : (b > L ? L : b);
    } else if (owner_short >= 0) {
      lo = c <= owner_short ? 0 : L;
      hi = c < owner_short ? 0 : L;
    } else {
      lo = chunk_lo(L, sp, c);
      hi = lo + chunk_len(L, sp, c);
    }
  }
  // tokens SP rank k holds of this sequence
  __device__ __forceinline__ int64_t held(int k) const {
    int64_t lo, hi;
    bounds(k, lo, hi);
    int64_t n = hi - lo;
    if (split == EARL_SP_ZIGZAG) {
      bounds(2 * sp - 1 - k, lo, hi);
      n += hi - lo;
    }
    return n;
  }
};

__device__ __forceinline__ Chunker make_chunker(const PlanArgs& a, int l, int64_t i,
                                                const int64_t* group_tokens) {
  const LayoutDesc& D = a.lay[l];
  Chunker c;
  c.split = D.split;
  c.sp = D.sp;
  c.C = D.split == EARL_SP_ZIGZAG ? 2 * D.sp : D.sp;
  c.L = a.lens[i];
  c.gpos = 0;
  c.S = 0;
  c.owner_short = -1;
  if (D.split == EARL_SP_FLAT) {
    c.gpos = a.gpos[l][i];
    c.S = group_tokens[a.grp[l][i]];
  } else if (D.split == EARL_SP_THRESHOLD && c.L < D.min_len) {
    c.owner_short = a.pos[l][i] % D.sp;
  }
  return c;
}

// Two-pointer intersection of two chunkings of [0, L): calls f(cs, cd, x, y) for every
// non-empty overlap in increasing x.
template <class F>
__device__ __forceinline__ int for_each_piece(const Chunker& cs, const Chunker& cd, F f) {
  int p = 0, q = 0, cnt = 0;
  while (p < cs.C && q < cd.C) {
    int64_t as, bs, ad, bd;
    cs.bounds(p, as, bs);
    cd.bounds(q, ad, bd);
    const int64_t x = as > ad ? as : ad, y = bs < bd ? bs : bd;
    if (x < y) { f(p, q, x, y); ++cnt; }
    if (bs < bd) ++p;
    else if (bd < bs) ++q;
    else { ++p; ++q; }
  }
  return cnt;
}

// LPT (one CTA; N <= 8192): bitonic sort of (INT32_MAX - L, i) keys in shared memory, then
// Graham's greedy in one thread with the D <= 8 loads in registers.
__device__ __noinline__ void lpt_assign(const PlanArgs& a, int l, uint64_t* keys) {
  const int tid = threadIdx.x;
  const int64_t N = a.N;
  const int D = a.lay[l].dp;
  int64_t n2 = 1;
  while (n2 < N) n2 <<= 1;
  for (int64_t i = tid; i < n2; i += NT)
    keys[i] = (i < N) ? ((uint64_t)(0x7fffffffu - (uint32_t)a.lens[i]) << 32) | (uint64_t)i
                      : ~0ull;
  __syncthreads();
  for (int64_t k = 2; k <= n2; k <<= 1) {
    for (int64_t j = k >> 1; j > 0; j >>= 1) {
      for (int64_t i = tid; i < n2; i += NT) {
        const int64_t ixj = i ^ j;
        if (ixj > i) {
          const uint64_t x = keys[i], y = keys[ixj];
          const bool asc = (i & k) == 0;
          if ((x > y) == asc) { keys[i] = y; keys[ixj] = x; }
        }
      }
      __syncthreads();
    }
  }
  if (a.P[N] < (1LL << 28)) {
    // Graham's greedy on warp 0: lane g holds group g's load; the least-loaded group (ties to
    // the lowest index) is one __reduce_min_sync over (load << 3 | g) -- loads stay < 2^28
    if (tid < 32) {
      const int lane = tid;
      uint32_t load = 0;
      for (int64_t q = 0; q < N; ++q) {
        const uint64_t key = keys[q];
        const uint32_t L = 0x7fffffffu - (uint32_t)(key >> 32);
        const uint32_t packed = lane < D ? ((load << 3) | (uint32_t)lane) : 0xffffffffu;
        const uint32_t m = __reduce_min_sync(kFull, packed);
        const int best = (int)(m & 7u);
        if (lane == best) load += L;
        __syncwarp();
        if (lane == 0) keys[q] = (key & 0xffffffffull) | ((uint64_t)best << 32);
      }
    }
  } else if (tid == 0) {
    // Graham's greedy: the least-loaded group (ties to the lowest index) by a depth-3
    // tournament over the <= 8 register-resident loads (groups >= D never win)
    int64_t ld[kMaxShards];
#pragma unroll
    for (int g = 0; g < kMaxShards; ++g) ld[g] = g < D ? 0 : INT64_MAX;
    constexpr int kB = 8;  // keys are read 8 at a time (independent loads off the chain)
    for (int64_t q0 = 0; q0 < N; q0 += kB) {
      uint64_t kb[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) kb[u] = (q0 + u < N) ? keys[q0 + u] : 0;
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        if (q0 + u >= N) break;
        const int64_t L = (int64_t)(0x7fffffffu - (uint32_t)(kb[u] >> 32));
        int w1[4];
        int64_t v1[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const bool right = ld[2 * p + 1] < ld[2 * p];
          w1[p] = right ? 2 * p + 1 : 2 * p;
          v1[p] = right ? ld[2 * p + 1] : ld[2 * p];
        }
        const bool r2a = v1[1] < v1[0], r2b = v1[3] < v1[2];
        const int wa = r2a ? w1[1] : w1[0], wb = r2b ? w1[3] : w1[2];
        const int64_t va = r2a ? v1[1] : v1[0], vb = r2b ? v1[3] : v1[2];
        const int best = vb < va ? wb : wa;
#pragma unroll
        for (int g = 0; g < kMaxShards; ++g)
          if (g == best) ld[g] += L;
        // the key is consumed: keep (i, group) in its slot for the parallel write-out
        keys[q0 + u] = (kb[u] & 0xffffffffull) | ((uint64_t)best << 32);
      }
    }
  }
  __syncthreads();
  for (int64_t q = tid; q < N; q += NT) {
    const uint64_t v = keys[q];
    a.grp[l][(int)(v & 0xffffffffu)] = (int32_t)(v >> 32);
  }
  __syncthreads();
}

// Per-(rank, dst shard) record / token bases and message byte offsets from the per-key piece
// starts kstart[0..K] and token totals ktok[K] (key = src shard * Sd + dst shard).  Every CTA
// derives them in shared memory (warp 0, two entries per lane, warp scans); CTA 0 publishes them
// in the header for the copy kernels and the host, and writes the records' token-prefix sentinel.
struct Tables {
  int64_t rbase[kMaxWorld][kMaxShards], tbase[kMaxWorld][kMaxShards];
  int64_t rec_begin[kMaxWorld + 1], tok_begin[kMaxWorld + 1];
  int64_t msg_off[kMaxKeys], stage[kMaxShards], msgb[kMaxKeys];
};

__device__ __noinline__ void build_tables(const PlanArgs& a, int K, const int64_t* kstart,
                                          const int64_t* ktok, Tables& tb) {
  const int tid = threadIdx.x;
  const LayoutDesc& S = a.lay[0];
  const LayoutDesc& Dl = a.lay[1];
  const int Sd = Dl.dp * Dl.sp;
  const int nts = S.tp < Dl.tp ? S.tp : Dl.tp;
  PlanHeader* h = a.hdr;
  if (tid < 32) {
    const int lane = tid;
    const int E = a.world * Sd;
    int64_t cnt[2], tk[2];
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
      const int e = lane + 32 * hf;
      cnt[hf] = 0;
      tk[hf] = 0;
      if (e < E) {
        const int r = e / Sd, ds = e - (e / Sd) * Sd;
        const int rr = r - S.rank0;
        if (rr >= 0 && rr < S.dp * S.sp * S.tp && rr % S.tp < nts) {
          const int key = (rr / S.tp) * Sd + ds;
          cnt[hf] = kstart[key + 1] - kstart[key];
          tk[hf] = ktok[key];
        }
      }
    }
    int64_t carry_c = 0, carry_t = 0;
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
      int64_t ic = cnt[hf], it = tk[hf];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t yc = __shfl_up_sync(kFull, ic, o), yt = __shfl_up_sync(kFull, it, o);
        if (lane >= o) { ic += yc; it += yt; }
      }
      const int e = lane + 32 * hf;
      if (e < E) {
        const int r = e / Sd, ds = e - (e / Sd) * Sd;
        tb.rbase[r][ds] = carry_c + ic - cnt[hf];
        tb.tbase[r][ds] = carry_t + it - tk[hf];
        if (ds == 0) { tb.rec_begin[r] = tb.rbase[r][0]; tb.tok_begin[r] = tb.tbase[r][0]; }
      }
      carry_c += __shfl_sync(kFull, ic, 31);
      carry_t += __shfl_sync(kFull, it, 31);
    }
    if (lane == 0) { tb.rec_begin[a.world] = carry_c; tb.tok_begin[a.world] = carry_t; }
    // message bytes per key, then the offset of each message inside its source shard's buffer
    for (int key = lane; key < K; key += 32) {
      int64_t mb = 0;
      for (int f = 0; f < a.n_fields; ++f) mb += (ktok[key] * a.Bf[f] + 15) & ~15LL;
      tb.msgb[key] = mb;
    }
    __syncwarp();
    for (int key = lane; key < K; key += 32) {
      const int ss = key / Sd, ds = key - ss * Sd;
      int64_t off = 0;
      for (int q = 0; q < ds; ++q) off += tb.msgb[ss * Sd + q];
      tb.msg_off[key] = off;
      if (ds == Sd - 1) tb.stage[ss] = off + tb.msgb[key];
    }
  }
  __syncthreads();
  if (blockIdx.x == 0) {
    if (tid <= K) h->key_piece_start[tid] = kstart[tid];
    if (tid < K) {
      h->key_pieces[tid] = kstart[tid + 1] - kstart[tid];
      h->key_tokens[tid] = ktok[tid];
      h->msg_off[tid] = tb.msg_off[tid];
    }
    if (tid < S.dp * S.sp) h->stage_bytes_shard[tid] = tb.stage[tid];
    if (tid <= a.world) {
      h->rec_begin[tid] = tb.rec_begin[tid];
      h->rec_tok_begin[tid] = tb.tok_begin[tid];
    }
    if (tid < a.world * Sd) {
      h->rec_base[tid / Sd][tid % Sd] = tb.rbase[tid / Sd][tid % Sd];
      h->rec_tok_base[tid / Sd][tid % Sd] = tb.tbase[tid / Sd][tid % Sd];
    }
    if (tid == 0) {
      h->n_records = tb.rec_begin[a.world];
      h->rec_tokens = tb.tok_begin[a.world];
      a.rec.tok_prefix[tb.rec_begin[a.world]] = tb.tok_begin[a.world];
    }
  }
}

__global__ void __launch_bounds__(NT, 1) planner_kernel(const __grid_constant__ PlanArgs a) {
  extern __shared__ uint64_t lpt_keys[];
  __shared__ int64_t sm_scan[NT / 32 + 1];
  __shared__ PartitionSmem ps;
  PlanHeader* h = a.hdr;
  const int tid = threadIdx.x;
  const bool lead = blockIdx.x == 0;
  const int64_t N = a.N;
  const int64_t gtid = (int64_t)blockIdx.x * NT + tid, gstride = (int64_t)gridDim.x * NT;

  // ---- phase 0: lengths, P, T -------------------------------------------------------
  stamp(a, 0);
  __shared__ unsigned s_max;
  if (tid == 0) s_max = 0;
  __syncthreads();
  uint32_t lmax = 0;
  for (int64_t i = gtid; i < N; i += gstride) {
    int32_t L = a.seq_lens[i];
    if (L < 0) { latch(h, EARL_ERR_INVALID_ARGUMENT, (int)i); L = 0; }
    a.lens[i] = L;
    a.vtmp[i] = L;
    lmax = max(lmax, (uint32_t)L);
  }
  publish_max_len(h, lmax, &s_max);
  gsync();
  const int64_t T = scan_array(a.vtmp, a.P, N, a.cta_sums, sm_scan);
  if (lead && tid == 0) { a.P[N] = T; h->T = T; }
  gsync();

  // ---- phase 1: assignment -----------------------------------------------------------
  stamp(a, 1);
  for (int l = 0; l < 2; ++l) {
    const LayoutDesc& L = a.lay[l];
    const int D = L.dp;
    if (L.assign == EARL_ASSIGN_LPT) {
      if (lead) lpt_assign(a, l, lpt_keys);
      continue;
    }
    // GIVEN_COUNTS and CONTIG groups are monotone in i: their starts are published here and
    // phase 2 needs no partition for them
    if (L.assign == EARL_ASSIGN_GIVEN_COUNTS && lead && tid <= D)
      h->group_start[l][tid] = L.count_start[tid];
    auto contig = [&](int64_t i) -> int {
      if (T == 0) {  // count blocks, earlier groups take the extra
        const int64_t q = N / D, r = N % D;
        return (i < r * (q + 1)) ? (int)(i / (q + 1)) : (int)(r + (i - r * (q + 1)) / q);
      }
      const int64_t m = ((int64_t)D * (2 * a.P[i] + a.lens[i])) / (2 * T);
      return (int)(m < D - 1 ? m : D - 1);
    };
    for (int64_t i = gtid; i < N; i += gstride) {
      int g = 0;
      if (L.assign == EARL_ASSIGN_GIVEN_COUNTS) {
        while (g < D - 1 && i >= L.count_start[g + 1]) ++g;
      } else if (L.assign == EARL_ASSIGN_CONTIG) {
        g = contig(i);
        const int gp = i > 0 ? contig(i - 1) : -1;  // groups gp+1 .. g start at i
        for (int k = gp + 1; k <= g; ++k) h->group_start[l][k] = i;
        if (i == N - 1)
          for (int k = g + 1; k <= D; ++k) h->group_start[l][k] = N;
      } else {  // EXPLICIT
        g = L.group_of_seq[i];
        if (g < 0 || g >= D) { latch(h, EARL_ERR_LAYOUT, (int)i); g = 0; }
      }
      a.grp[l][i] = g;
    }
  }
  gsync();

  // ---- phase 2: per-layout group order and local token offsets ------------------------
  stamp(a, 2);
  __shared__ int64_t s_gtok[2][kMaxShards];
  __shared__ int64_t s_gstart[kMaxShards + 1];
  for (int l = 0; l < 2; ++l) {
    const LayoutDesc& L = a.lay[l];
    const int D = L.dp, SP = L.sp;
    const int32_t* grp = a.grp[l];
    int32_t* perm = a.perm[l];
    // monotone groups (GIVEN_COUNTS, CONTIG): the stable partition by group is the identity
    // and every per-sequence value below is written and first read by the same thread
    const bool mono = L.assign == EARL_ASSIGN_GIVEN_COUNTS || L.assign == EARL_ASSIGN_CONTIG;
    if (mono) {
      for (int64_t j = gtid; j < N; j += gstride) perm[j] = (int32_t)j;
      if (tid <= D) s_gstart[tid] = __ldcg(&h->group_start[l][tid]);  // phase 1 (other CTAs)
      __syncthreads();
    } else {
      partition_array(grp, N, D, perm, a.ghist, ps);
      if (lead && tid <= D) h->group_start[l][tid] = ps.bstart[tid];
      if (tid <= D) s_gstart[tid] = ps.bstart[tid];
      gsync();
    }
    stamp(a, 10 + 3 * l);
    if (lead && tid < D) h->group_count[l][tid] = s_gstart[tid + 1] - s_gstart[tid];
    if (L.split == EARL_SP_FLAT || L.split == EARL_SP_THRESHOLD) {
      // position of every sequence in its group, and its offset in the group's token stream
      if (mono) {  // the group streams are slices of P
        for (int64_t j = gtid; j < N; j += gstride) {
          const int64_t s0 = s_gstart[grp[j]];
          a.pos[l][j] = (int32_t)(j - s0);
          a.gpos[l][j] = a.P[j] - a.P[s0];
        }
        if (tid < D) s_gtok[l][tid] = a.P[s_gstart[tid + 1]] - a.P[s_gstart[tid]];
        __syncthreads();
      } else {
        int64_t* cum0 = a.cum[l];
        for (int64_t j = gtid; j < N; j += gstride) {
          const int i = perm[j];
          a.pos[l][i] = (int32_t)(j - s_gstart[grp[i]]);
          a.vtmp[j] = a.lens[i];
        }
        gsync();
        const int64_t tot = scan_array(a.vtmp, cum0, N, a.cta_sums, sm_scan);
        if (lead && tid == 0) cum0[N] = tot;
        gsync();
        for (int64_t j = gtid; j < N; j += gstride) {
          const int i = perm[j];
          a.gpos[l][i] = cum0[j] - cum0[s_gstart[grp[i]]];
        }
        if (tid < D) s_gtok[l][tid] = cum0[s_gstart[tid + 1]] - cum0[s_gstart[tid]];
        gsync();
      }
    } else if (tid < D) {
      s_gtok[l][tid] = 0;
    }
    if (lead && tid < D) h->group_tokens[l][tid] = s_gtok[l][tid];
    stamp(a, 11 + 3 * l);
    if (mono && SP == 1) {
      // one chunk holding the whole sequence, in index order: the chunk scan is P itself
      int64_t* cum = a.cum[l];
      int64_t* off = a.off[l];
      for (int64_t j = gtid; j <= N; j += gstride) {
        cum[j] = a.P[j];
        if (j < N) off[j] = a.P[j] - a.P[s_gstart[grp[j]]];
      }
      if (lead && tid < D) {
        const int64_t st = a.P[s_gstart[tid + 1]] - a.P[s_gstart[tid]];
        h->shard_tokens[l][tid] = st;
        if (l == 1 && st > 0x7fffffffLL) latch(h, EARL_ERR_CAPACITY, tid);
      }
    } else {
      for (int k = 0; k < SP; ++k) {
        int64_t* cum = a.cum[l] + (int64_t)k * (N + 1);
        int64_t* off = a.off[l] + (int64_t)k * N;
        for (int64_t j = gtid; j < N; j += gstride)
          a.vtmp[j] = make_chunker(a, l, perm[j], s_gtok[l]).held(k);
        gsync();
        const int64_t tot = scan_array(a.vtmp, cum, N, a.cta_sums, sm_scan);
        if (lead && tid == 0) cum[N] = tot;
        gsync();
        for (int64_t j = gtid; j < N; j += gstride) {
          const int i = perm[j];
          off[i] = cum[j] - cum[s_gstart[grp[i]]];
        }
        if (lead && tid < D) {
          const int64_t st = cum[s_gstart[tid + 1]] - cum[s_gstart[tid]];
          h->shard_tokens[l][tid * SP + k] = st;
          if (l == 1 && st > 0x7fffffffLL) latch(h, EARL_ERR_CAPACITY, tid * SP + k);
        }
        // the next scan begins with a barrier-free read of lens/perm only; off and
        // shard_tokens are consumed after later barriers
      }
    }
    stamp(a, 12 + 3 * l);
    gsync();
  }

  // ---- phase 3: pieces ----------------------------------------------------------------
  stamp(a, 3);
  const LayoutDesc& S = a.lay[0];
  const LayoutDesc& Dl = a.lay[1];
  const int Sd = Dl.dp * Dl.sp;
  for (int64_t i = gtid; i < N; i += gstride)
    a.vtmp[i] = for_each_piece(make_chunker(a, 0, i, s_gtok[0]), make_chunker(a, 1, i, s_gtok[1]),
                               [](int, int, int64_t, int64_t) {});
  gsync();
  const int64_t M = scan_array(a.vtmp, a.pbase, N, a.cta_sums, sm_scan);
  if (lead && tid == 0) { a.pbase[N] = M; h->n_pieces = M; }
  gsync();
  for (int64_t i = gtid; i < N; i += gstride) {
    int64_t p = a.pbase[i];
    const int ss0 = a.grp[0][i] * S.sp, ds0 = a.grp[1][i] * Dl.sp;
    const Chunker ch_s = make_chunker(a, 0, i, s_gtok[0]), ch_d = make_chunker(a, 1, i, s_gtok[1]);
    for_each_piece(ch_s, ch_d, [&](int cs, int cd, int64_t x, int64_t y) {
      const int key = (ss0 + ch_s.owner(cs)) * Sd + ds0 + ch_d.owner(cd);
      a.pc_i[p] = (int32_t)i;
      a.pc_x[p] = (int32_t)x;
      a.pc_y[p] = (int32_t)y;
      a.pc_kk[p] = cs | (cd << 8) | (key << 16);
      a.ktmp[p] = key;
      ++p;
    });
  }
  gsync();

  // ---- phase 4: pieces by message key, message token offsets -------------------------
  stamp(a, 4);
  const int K = S.dp * S.sp * Sd;
  partition_array(a.ktmp, M, K, a.ptmp, a.ghist, ps);
  __shared__ int64_t s_kstart[kMaxKeys + 1], s_ktok[kMaxKeys], s_kscan0[kMaxKeys];
  if (tid <= K) s_kstart[tid] = ps.bstart[tid];
  gsync();
  for (int64_t pos = gtid; pos < M; pos += gstride) {
    const int32_t q = a.ptmp[pos];
    a.ps_i[pos] = a.pc_i[q];
    a.ps_x[pos] = a.pc_x[q];
    a.ps_y[pos] = a.pc_y[q];
    a.ps_kk[pos] = a.pc_kk[q];
    a.vtmp[pos] = a.pc_y[q] - a.pc_x[q];
  }
  gsync();
  const int64_t Mtok = scan_array(a.vtmp, a.ps_scan, M, a.cta_sums, sm_scan);
  if (lead && tid == 0) a.ps_scan[M] = Mtok;
  gsync();

  // ---- phase 5: bases and message offsets ---------------------------------------------
  stamp(a, 5);
  // Every CTA derives the <= 64-entry tables itself in shared memory (parallel loads of the
  // published scan, then warp 0 scans <= 64 entries); CTA 0 also publishes them in the header
  // for the copy kernels and the host.
  const int nts = S.tp < Dl.tp ? S.tp : Dl.tp;
  if (tid < K) {
    s_kscan0[tid] = a.ps_scan[s_kstart[tid]];
    s_ktok[tid] = a.ps_scan[s_kstart[tid + 1]] - s_kscan0[tid];
  }
  __syncthreads();
  stamp(a, 8);
  __shared__ Tables tb;
  build_tables(a, K, s_kstart, s_ktok, tb);
  stamp(a, 9);

  // ---- phase 6: records ---------------------------------------------------------------
  stamp(a, 6);
  const int64_t nrec = M * nts;
  for (int64_t idx = gtid; idx < nrec; idx += gstride) {
    const int64_t q = idx / nts;
    const int ts = (int)(idx - q * nts);
    const int kk = a.ps_kk[q];
    const int ks = kk & 0xff, kd = (kk >> 8) & 0xff, key = kk >> 16;
    const int ss = key / Sd, ds = key - ss * Sd;
    const int s = S.rank0 + ss * S.tp + ts;
    const int64_t rho = q - s_kstart[key];
    const int64_t j = tb.rbase[s][ds] + rho;
    const int i = a.ps_i[q];
    const int64_t x = a.ps_x[q], y = a.ps_y[q];
    const int64_t msg_tok = a.ps_scan[q] - s_kscan0[key];
    a.rec.seq[j] = i;
    a.rec.x[j] = (int32_t)x;
    a.rec.n[j] = (int32_t)(y - x);
    a.rec.code[j] = (uint32_t)s | ((uint32_t)ss << 8) | ((uint32_t)ds << 16) | ((uint32_t)ts << 24);
    {
      // local offset of virtual chunk c = offset of the sequence's holding on SP rank owner(c)
      // (+ the first chunk's length for ZIGZAG's second chunk)
      const Chunker ch_s = make_chunker(a, 0, i, s_gtok[0]), ch_d = make_chunker(a, 1, i, s_gtok[1]);
      int64_t lo, hi, lo0, hi0;
      const int os = ch_s.owner(ks), od = ch_d.owner(kd);
      ch_s.bounds(ks, lo, hi);
      int64_t so = a.off[0][(int64_t)os * N + i] + (x - lo);
      if (ks != os) { ch_s.bounds(os, lo0, hi0); so += hi0 - lo0; }
      ch_d.bounds(kd, lo, hi);
      int64_t dof = a.off[1][(int64_t)od * N + i] + (x - lo);
      if (kd != od) { ch_d.bounds(od, lo0, hi0); dof += hi0 - lo0; }
      a.rec.src_tok[j] = so;
      a.rec.dst_tok[j] = dof;
    }
    a.rec.msg_tok[j] = msg_tok;
    a.rec.tok_prefix[j] = tb.tbase[s][ds] + msg_tok;
  }
  stamp(a, 7);
}

// ---------------------------------------------------------------------------------------
// SP = 1 fast path.  When neither layout splits sequences (sp == 1 on both sides, any
// assignment), a piece is a whole sequence with L > 0 and every plan array is a stable
// per-bucket rank or token prefix over three bucketings of the sequences: by message key
// (src group, dst group; pieces only), by src group and by dst group (every sequence).  One
// kernel computes them all with two grid barriers (three with LPT) instead of the general
// path's ~20: each CTA owns a contiguous tile of sequences, histograms its buckets, and after
// one barrier emits every output from (CTAs before it) + (chunks before) + (warps before) +
// (lanes before).  Same outputs, bit for bit, as the general planner (tested against it and
// against the oracle).
// ---------------------------------------------------------------------------------------

constexpr int kMaxBuckets = kMaxKeys + 2 * kMaxShards;

struct FastSmem {
  int32_t wcnt[NT / 32][kMaxBuckets];  // per-warp bucket counts of a chunk, then exclusive over warps
  int64_t wtok[NT / 32][kMaxBuckets];
  int64_t run_cnt[kMaxBuckets], run_tok[kMaxBuckets];      // before the current chunk
  int64_t chunk_cnt[kMaxBuckets], chunk_tok[kMaxBuckets];  // the current chunk's totals
  int64_t tot_cnt[kMaxBuckets], tot_tok[kMaxBuckets];      // whole batch
  unsigned long long hcnt[kMaxBuckets], htok[kMaxBuckets];  // this CTA's histogram
  int64_t gstart[2][kMaxShards + 1], gtok0[2][kMaxShards + 1];
  int64_t kstart[kMaxKeys + 1], ktok[kMaxKeys];
  int64_t carry, total;
};

// The calling lane's bucket u (-1: none) with weight L: its rank among the warp's lanes below
// it in the same bucket, the token prefix over them, and -- on the highest lane of each bucket --
// the bucket's warp count and tokens.  The token prefix runs one warp scan per distinct bucket
// of the warp (1 for layouts that keep neighbours together, <= 8 for a round-robin one).
__device__ __forceinline__ void warp_bucket(int u, int64_t L, int lane, int& rank, int64_t& tpre,
                                            bool& last, int& gcnt, int64_t& gtok) {
  const unsigned peers = __match_any_sync(kFull, u);
  rank = __popc(peers & ((1u << lane) - 1u));
  gcnt = __popc(peers);
  last = (31 - __clz(peers)) == lane;
  tpre = 0;
  gtok = 0;
  unsigned rem = kFull;
  while (rem) {
    const int leader = __ffs(rem) - 1;
    const int ub = __shfl_sync(kFull, u, leader);
    const bool mine = u == ub;
    const unsigned m = __ballot_sync(kFull, mine);
    int64_t v = mine ? L : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(kFull, v, o);
      if (lane >= o) v += y;
    }
    if (mine) { tpre = v - L; gtok = v; }
    rem &= ~m;
  }
}

__device__ __forceinline__ int assign_group(const PlanArgs& a, const LayoutDesc& Ly, PlanHeader* h,
                                            int64_t i, int64_t L, int64_t Pi, int64_t T, int64_t N) {
  const int D = Ly.dp;
  int g = 0;
  if (Ly.assign == EARL_ASSIGN_GIVEN_COUNTS) {
    while (g < D - 1 && i >= Ly.count_start[g + 1]) ++g;
  } else if (Ly.assign == EARL_ASSIGN_CONTIG) {
    if (T == 0) {
      const int64_t q = N / D, r = N % D;
      g = (i < r * (q + 1)) ? (int)(i / (q + 1)) : (int)(r + (i - r * (q + 1)) / q);
    } else {
      const int64_t m = ((int64_t)D * (2 * Pi + L)) / (2 * T);
      g = (int)(m < D - 1 ? m : D - 1);
    }
  } else {  // EXPLICIT
    g = Ly.group_of_seq[i];
    if (g < 0 || g >= D) { latch(h, EARL_ERR_LAYOUT, (int)i); g = 0; }
  }
  return g;
}

__global__ void __launch_bounds__(NT, 1) planner_sp1_kernel(const __grid_constant__ PlanArgs a) {
  extern __shared__ uint64_t lpt_keys[];
  __shared__ int64_t sm_scan[NT / 32 + 1];
  __shared__ FastSmem fs;
  __shared__ Tables tb;
  PlanHeader* h = a.hdr;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const bool lead = blockIdx.x == 0;
  const int64_t N = a.N;
  const int64_t lo = range_lo(N), hi = range_hi(N);
  const int nchunks = (int)((hi - lo + NT - 1) / NT);
  const LayoutDesc& S = a.lay[0];
  const LayoutDesc& Dl = a.lay[1];
  const int Ds = S.dp, Dd = Dl.dp;
  const int K = Ds * Dd;
  const int U = K + Ds + Dd;
  const bool lpt = S.assign == EARL_ASSIGN_LPT || Dl.assign == EARL_ASSIGN_LPT;

  // ---- lengths, the CTA's token sum; P and T after one barrier ------------------------
  stamp(a, 0);
  __shared__ unsigned s_max;
  if (tid == 0) s_max = 0;
  __syncthreads();
  int64_t part = 0;
  uint32_t lmax = 0;
  for (int c = 0; c < nchunks; ++c) {
    const int64_t i = lo + (int64_t)c * NT + tid;
    if (i < hi) {
      int32_t L = a.seq_lens[i];
      if (L < 0) { latch(h, EARL_ERR_INVALID_ARGUMENT, (int)i); L = 0; }
      a.lens[i] = L;
      part += L;
      lmax = max(lmax, (uint32_t)L);
    }
  }
  publish_max_len(h, lmax, &s_max);
  {
    int64_t tot;
    block_excl_scan(part, tot, sm_scan);
    if (tid == 0) a.cta_sums[blockIdx.x] = tot;
  }
  if (tid < kMaxBuckets) {
    fs.hcnt[tid] = 0; fs.htok[tid] = 0;
    fs.run_cnt[tid] = 0; fs.tot_cnt[tid] = 0; fs.run_tok[tid] = 0; fs.tot_tok[tid] = 0;
  }
  gsync();
  if (tid < 32) {
    int64_t before = 0, all = 0;
    for (int b = tid; b < (int)gridDim.x; b += 32) {
      const int64_t v = __ldcg(&a.cta_sums[b]);
      all += v;
      if (b < (int)blockIdx.x) before += v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      before += __shfl_xor_sync(kFull, before, o);
      all += __shfl_xor_sync(kFull, all, o);
    }
    if (tid == 0) { fs.carry = before; fs.total = all; }
  }
  __syncthreads();
  const int64_t T = fs.total;
  stamp(a, 1);
  {
    int64_t run = fs.carry;
    for (int c = 0; c < nchunks; ++c) {
      const int64_t i = lo + (int64_t)c * NT + tid;
      const int64_t L = i < hi ? a.lens[i] : 0;
      int64_t tot;
      const int64_t ex = run + block_excl_scan(L, tot, sm_scan);
      if (i < hi) {
        a.P[i] = ex;
        // assignment (LPT below, in CTA 0)
        if (S.assign != EARL_ASSIGN_LPT) a.grp[0][i] = assign_group(a, S, h, i, L, ex, T, N);
        if (Dl.assign != EARL_ASSIGN_LPT) a.grp[1][i] = assign_group(a, Dl, h, i, L, ex, T, N);
      }
      run += tot;
    }
  }
  if (lead && tid == 0) { a.P[N] = T; h->T = T; }
  if (lpt) {
    __syncthreads();
    if (lead) {
      if (S.assign == EARL_ASSIGN_LPT) lpt_assign(a, 0, lpt_keys);
      if (Dl.assign == EARL_ASSIGN_LPT) lpt_assign(a, 1, lpt_keys);
    }
    gsync();
  }

  // ---- this CTA's bucket histograms, published; totals and bases after one barrier ------
  stamp(a, 2);
  for (int c = 0; c < nchunks; ++c) {
    const int64_t i = lo + (int64_t)c * NT + tid;
    const bool ok = i < hi;
    const int64_t L = ok ? a.lens[i] : 0;
    const int gs = ok ? __ldcg(&a.grp[0][i]) : 0, gd = ok ? __ldcg(&a.grp[1][i]) : 0;
    const int ub[3] = {ok && L > 0 ? gs * Dd + gd : -1, ok ? K + gs : -1, ok ? K + Ds + gd : -1};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      int rank, gcnt;
      int64_t tpre, gtok;
      bool last;
      warp_bucket(ub[k], L, lane, rank, tpre, last, gcnt, gtok);
      if (last && ub[k] >= 0) {
        atomicAdd(&fs.hcnt[ub[k]], (unsigned long long)gcnt);
        atomicAdd(&fs.htok[ub[k]], (unsigned long long)gtok);
      }
    }
  }
  __syncthreads();
  int64_t* fh = a.fhist;  // [2][gridDim.x][kMaxBuckets]: counts, then tokens
  if (tid < U) {
    fh[(int64_t)blockIdx.x * kMaxBuckets + tid] = (int64_t)fs.hcnt[tid];
    fh[((int64_t)gridDim.x + blockIdx.x) * kMaxBuckets + tid] = (int64_t)fs.htok[tid];
  }
  gsync();
  stamp(a, 3);
  // per bucket: the sum over the CTAs before this one and over all.  The whole CTA reads the
  // published histograms at once: thread t sums column t % 2U (counts, then tokens) over the
  // CTAs r, r + R, ... (r = t / 2U, R = NT / 2U), loads unrolled, then one shared-memory atomic
  // per thread (a warp per column had put one L2 round trip per column on the critical path).
  {
    const int Q = 2 * U;
    const int R = NT / Q;
    const int G = (int)gridDim.x;
    if (tid < Q * R) {
      const int q = tid % Q, r0 = tid / Q;
      const int u = q < U ? q : q - U;
      const int64_t* col = fh + (q < U ? 0 : (int64_t)G * kMaxBuckets) + u;
      int64_t before = 0, all = 0;
#pragma unroll 4
      for (int b = r0; b < G; b += R) {
        const int64_t x = __ldcg(col + (int64_t)b * kMaxBuckets);
        all += x;
        if (b < (int)blockIdx.x) before += x;
      }
      if (q < U) {
        atomicAdd(reinterpret_cast<unsigned long long*>(&fs.run_cnt[u]), (unsigned long long)before);
        atomicAdd(reinterpret_cast<unsigned long long*>(&fs.tot_cnt[u]), (unsigned long long)all);
      } else {
        atomicAdd(reinterpret_cast<unsigned long long*>(&fs.run_tok[u]), (unsigned long long)before);
        atomicAdd(reinterpret_cast<unsigned long long*>(&fs.tot_tok[u]), (unsigned long long)all);
      }
    }
  }
  __syncthreads();
  // bases: group starts (sequence positions and tokens) per layout, message keys
  if (tid == 0) {
    for (int l = 0; l < 2; ++l) {
      const int D = l ? Dd : Ds, b0 = l ? K + Ds : K;
      int64_t cs = 0, ts = 0;
      for (int g = 0; g < D; ++g) {
        fs.gstart[l][g] = cs; fs.gtok0[l][g] = ts;
        cs += fs.tot_cnt[b0 + g]; ts += fs.tot_tok[b0 + g];
      }
      fs.gstart[l][D] = cs; fs.gtok0[l][D] = ts;
    }
    int64_t ks = 0;
    for (int k = 0; k < K; ++k) { fs.kstart[k] = ks; fs.ktok[k] = fs.tot_tok[k]; ks += fs.tot_cnt[k]; }
    fs.kstart[K] = ks;
  }
  __syncthreads();
  if (lead) {
    for (int l = 0; l < 2; ++l) {
      const LayoutDesc& Ly = a.lay[l];
      const int D = Ly.dp;
      if (tid <= D) h->group_start[l][tid] = fs.gstart[l][tid];
      if (tid < D) {
        const int64_t st = fs.gtok0[l][tid + 1] - fs.gtok0[l][tid];
        h->group_count[l][tid] = fs.gstart[l][tid + 1] - fs.gstart[l][tid];
        h->shard_tokens[l][tid] = st;
        h->group_tokens[l][tid] = (Ly.split == EARL_SP_FLAT || Ly.split == EARL_SP_THRESHOLD) ? st : 0;
        if (l == 1 && st > 0x7fffffffLL) latch(h, EARL_ERR_CAPACITY, tid);
      }
    }
    if (tid == 0) { h->n_pieces = fs.kstart[K]; a.cum[0][N] = T; a.cum[1][N] = T; a.pbase[N] = fs.kstart[K]; }
  }
  build_tables(a, K, fs.kstart, fs.ktok, tb);
  stamp(a, 4);

  // ---- emission, chunk by chunk in sequence order ---------------------------------------
  const int nts = S.tp < Dl.tp ? S.tp : Dl.tp;
  const bool pos_s = S.split == EARL_SP_FLAT || S.split == EARL_SP_THRESHOLD;
  const bool pos_d = Dl.split == EARL_SP_FLAT || Dl.split == EARL_SP_THRESHOLD;
  for (int c = 0; c < nchunks; ++c) {
    const int64_t i = lo + (int64_t)c * NT + tid;
    const bool ok = i < hi;
    const int64_t L = ok ? a.lens[i] : 0;
    const int gs = ok ? __ldcg(&a.grp[0][i]) : 0, gd = ok ? __ldcg(&a.grp[1][i]) : 0;
    const int ub[3] = {ok && L > 0 ? gs * Dd + gd : -1, ok ? K + gs : -1, ok ? K + Ds + gd : -1};
    for (int q = tid; q < (NT / 32) * kMaxBuckets; q += NT) {
      (&fs.wcnt[0][0])[q] = 0;
      (&fs.wtok[0][0])[q] = 0;
    }
    __syncthreads();
    int rk[3];
    int64_t tp[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      int gcnt;
      int64_t gtok;
      bool last;
      warp_bucket(ub[k], L, lane, rk[k], tp[k], last, gcnt, gtok);
      if (last && ub[k] >= 0) { fs.wcnt[w][ub[k]] = gcnt; fs.wtok[w][ub[k]] = gtok; }
    }
    __syncthreads();
    if (tid < U) {  // exclusive over warps, chunk totals
      int64_t ac = 0, at = 0;
      for (int ww = 0; ww < NT / 32; ++ww) {
        const int64_t cc = fs.wcnt[ww][tid], tt = fs.wtok[ww][tid];
        fs.wcnt[ww][tid] = (int32_t)ac;
        fs.wtok[ww][tid] = at;
        ac += cc;
        at += tt;
      }
      fs.chunk_cnt[tid] = ac;
      fs.chunk_tok[tid] = at;
    }
    __syncthreads();
    if (ok) {
      int64_t grank[3], gtp[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const int u = ub[k] < 0 ? 0 : ub[k];
        grank[k] = fs.run_cnt[u] + fs.wcnt[w][u] + rk[k];
        gtp[k] = fs.run_tok[u] + fs.wtok[w][u] + tp[k];
      }
      // layouts: sorted position, local offset, held-length scan
      const int64_t ps = fs.gstart[0][gs] + grank[1], pd = fs.gstart[1][gd] + grank[2];
      a.perm[0][ps] = (int32_t)i;
      a.perm[1][pd] = (int32_t)i;
      a.off[0][i] = gtp[1];
      a.off[1][i] = gtp[2];
      a.cum[0][ps] = fs.gtok0[0][gs] + gtp[1];
      a.cum[1][pd] = fs.gtok0[1][gd] + gtp[2];
      if (pos_s) { a.pos[0][i] = (int32_t)grank[1]; a.gpos[0][i] = gtp[1]; }
      if (pos_d) { a.pos[1][i] = (int32_t)grank[2]; a.gpos[1][i] = gtp[2]; }
      a.pbase[i] = L > 0 ? grank[0] : 0;  // (diagnostic: piece rank inside its key)
      if (L > 0) {
        const int key = ub[0];
        for (int ts = 0; ts < nts; ++ts) {
          const int s = S.rank0 + gs * S.tp + ts;
          const int64_t j = tb.rbase[s][gd] + grank[0];
          a.rec.seq[j] = (int32_t)i;
          a.rec.x[j] = 0;
          a.rec.n[j] = (int32_t)L;
          a.rec.code[j] = (uint32_t)s | ((uint32_t)gs << 8) | ((uint32_t)gd << 16) | ((uint32_t)ts << 24);
          a.rec.src_tok[j] = gtp[1];
          a.rec.dst_tok[j] = gtp[2];
          a.rec.msg_tok[j] = gtp[0];
          a.rec.tok_prefix[j] = tb.tbase[s][gd] + gtp[0];
        }
        (void)key;
      }
    }
    __syncthreads();
    if (tid < U) { fs.run_cnt[tid] += fs.chunk_cnt[tid]; fs.run_tok[tid] += fs.chunk_tok[tid]; }
  }
  stamp(a, 7);
}

// Destination metadata of dst shard (g, k): cu_seqlens (int32), seq_ids (int64), tok_start.
__global__ void local_meta_kernel(const __grid_constant__ PlanArgs a, int g, int k, int32_t* cu,
                                  int64_t* ids, int32_t* tok_start) {
  const PlanHeader* h = a.hdr;
  const int64_t N = a.N;
  const int64_t n = h->group_count[1][g];
  const int64_t gs = h->group_start[1][g];
  const int64_t* cum = a.cum[1] + (int64_t)k * (N + 1);
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j <= n;
       j += (int64_t)gridDim.x * blockDim.x) {
    if (cu) cu[j] = (int32_t)(cum[gs + j] - cum[gs]);
    if (j < n) {
      const int i = a.perm[1][gs + j];
      if (ids) ids[j] = i;
      if (tok_start) {
        int64_t lo, hi;
        make_chunker(a, 1, i, h->group_tokens[1]).bounds(k, lo, hi);
        tok_start[j] = (int32_t)lo;
      }
    }
  }
}

}  // namespace

// Grid size: one CTA per 4096 items (sequences or pieces), at most what can be co-resident.
// EARL_PLAN_GRID=<g> forces g (tests use it to check that the plan does not depend on G).
int planner_grid(int64_t n_seqs, int64_t max_pieces, int sm_count, size_t lpt_smem, bool fast) {
  static int per_sm = -1;
  static bool opted[64] = {}, opted_fast[64] = {};
  opt_in_dynamic_smem(planner_kernel, 64 * 1024, opted);
  opt_in_dynamic_smem(planner_sp1_kernel, 64 * 1024, opted_fast);
  if (per_sm < 0) {
    int p1 = 1, p2 = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p1, planner_kernel, NT, 64 * 1024) != cudaSuccess)
      p1 = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p2, planner_sp1_kernel, NT, 64 * 1024) != cudaSuccess)
      p2 = 1;
    (void)cudaGetLastError();
    per_sm = p1 < p2 ? p1 : p2;
    if (per_sm < 1) per_sm = 1;
  }
  const char* env = getenv("EARL_PLAN_GRID");
  const int forced = env ? atoi(env) : -1;
  const int64_t work = n_seqs > max_pieces ? n_seqs : max_pieces;
  // the fast path's phases are one elementwise pass each: one CTA per 1024 sequences (a chunk)
  int64_t g = forced > 0 ? forced : fast ? (n_seqs + 1023) / 1024 : (work + 4095) / 4096;
  const int64_t cap = (int64_t)sm_count * per_sm;
  if (g > cap) g = cap;
  if (g > kMaxPlanGrid) g = kMaxPlanGrid;
  if (g < 1) g = 1;
  (void)lpt_smem;
  return (int)g;
}

cudaError_t launch_planner(const PlanArgs& a, size_t lpt_smem, int grid, bool fast, cudaStream_t s) {
  static bool configured[64] = {}, configured_fast[64] = {};
  cudaError_t e = opt_in_dynamic_smem(planner_kernel, 64 * 1024, configured);
  if (e == cudaSuccess) e = opt_in_dynamic_smem(planner_sp1_kernel, 64 * 1024, configured_fast);
  if (e != cudaSuccess) return e;
  auto kern = fast ? planner_sp1_kernel : planner_kernel;
  if (grid == 1) {
    kern<<<1, NT, lpt_smem, s>>>(a);
    return cudaGetLastError();
  }
  void* args[] = {const_cast<PlanArgs*>(&a)};
  return cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(NT), args, lpt_smem, s);
}

cudaError_t launch_local_meta(const PlanArgs& a, int g, int k, int32_t* cu, int64_t* ids,
                              int32_t* tok_start, cudaStream_t s) {
  local_meta_kernel<<<64, 256, 0, s>>>(a, g, k, cu, ids, tok_start);
  return cudaGetLastError();
}

}  // namespace earl
