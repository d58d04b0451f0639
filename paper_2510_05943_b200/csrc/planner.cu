// planner.cu -- device-side dispatch planner.
//
// One CTA of 1024 threads computes the whole plan in phases separated by __syncthreads, so the
// plan needs no host synchronisation, no inter-CTA protocol and is bit-for-bit deterministic
// (every rank computes the identical plan from the identical lengths; integer arithmetic only).
// The planner is latency-bound integer work (a few µs at the configs' N <= 512); every scan
// walks tiles of 4096 items with a block-wide warp-shuffle scan and carries the running total.
//
// Phases ("adaptive to the current data distribution layout and parallelism
// configuration"; the steps follow SURVEY.md §8(c) and the readings in DESIGN.md):
//   0  P = exclusive scan of L (int64), T = sum L; latch L_i < 0 (reading c20)
//   1  g(i) for src and dst: GIVEN_COUNTS / CONTIG midpoint / LPT / EXPLICIT (reading c4)
//   2  per layout: stable partition of sequences by group (ascending i inside a group, c5);
//      per SP chunk k: scan of BLOCK chunk lengths in that order -> local token offsets (c7)
//   3  pieces: two-pointer intersection of the src and dst chunk partitions of every sequence
//   4  stable partition of pieces by message key (src shard, dst shard); message token offsets
//   5  per-(rank, shard) record / token bases, message byte offsets (16-B aligned field blocks)
//   6  records: piece x sending replica ts < min(TP_src, TP_dst) (reading c9), in (s, ds, i, x)
#include "earl_internal.cuh"

namespace earl {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int NT = kPlanThreads;
constexpr int kItems = 4;

__device__ __forceinline__ void latch(PlanHeader* h, int code, int detail) {
  if (atomicCAS(&h->err, 0, code) == 0) h->err_detail = detail;
}

// BLOCK rule: q = L / sp, r = L % sp, chunk k = [k*q + min(k,r), (k+1)*q + min(k+1,r)).
__device__ __forceinline__ int64_t chunk_lo(int64_t L, int sp, int k) {
  const int64_t q = L / sp, r = L % sp;
  return k * q + (k < r ? (int64_t)k : r);
}
__device__ __forceinline__ int64_t chunk_len(int64_t L, int sp, int k) {
  return L / sp + ((int64_t)k < L % sp ? 1 : 0);
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

// Exclusive scan over [0, n): put(i, sum_{j<i} get(j)); returns the total.
template <class Get, class Put>
__device__ int64_t tile_scan(int64_t n, Get get, Put put, int64_t* sm) {
  int64_t carry = 0;
  for (int64_t base = 0; base < n; base += (int64_t)NT * kItems) {
    int64_t v[kItems];
    int64_t tsum = 0;
    const int64_t i0 = base + (int64_t)threadIdx.x * kItems;
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      v[it] = (i0 + it < n) ? get(i0 + it) : 0;
      tsum += v[it];
    }
    int64_t total;
    int64_t run = carry + block_excl_scan(tsum, total, sm);
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      if (i0 + it < n) put(i0 + it, run);
      run += v[it];
    }
    carry += total;
  }
  return carry;
}

struct PartitionSmem {
  int32_t whist[NT / 32][kMaxKeys];
  int64_t running[kMaxKeys];
  int64_t tile_tot[kMaxKeys];
  int64_t bstart[kMaxKeys + 1];
  unsigned hist[kMaxKeys];
};

// Stable counting sort of [0, n) by key(i) in [0, K), K <= 64: emit(i, sorted position).
// On return ps.bstart[0..K] holds the bucket starts (bstart[K] = n).
template <class KeyF, class Emit>
__device__ void stable_partition(int64_t n, int K, KeyF key, Emit emit, PartitionSmem& ps) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid < kMaxKeys) { ps.hist[tid] = 0; ps.running[tid] = 0; }
  __syncthreads();
  for (int64_t i = tid; i < n; i += NT) atomicAdd(&ps.hist[key(i)], 1u);
  __syncthreads();
  if (tid == 0) {
    int64_t acc = 0;
    for (int k = 0; k < K; ++k) { ps.bstart[k] = acc; acc += ps.hist[k]; }
    ps.bstart[K] = acc;
  }
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t base = 0; base < n; base += NT) {
    const int64_t i = base + tid;
    const int k = (i < n) ? key(i) : -1;
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

// Two-pointer intersection of the BLOCK partitions of [0, L) into sps and spd chunks:
// calls f(ks, kd, x, y) for every non-empty overlap in increasing x.
template <class F>
__device__ __forceinline__ int for_each_piece(int64_t L, int sps, int spd, F f) {
  int ks = 0, kd = 0, cnt = 0;
  while (ks < sps && kd < spd) {
    const int64_t as = chunk_lo(L, sps, ks), bs = as + chunk_len(L, sps, ks);
    const int64_t ad = chunk_lo(L, spd, kd), bd = ad + chunk_len(L, spd, kd);
    const int64_t x = as > ad ? as : ad, y = bs < bd ? bs : bd;
    if (x < y) { f(ks, kd, x, y); ++cnt; }
    if (bs < bd) ++ks;
    else if (bd < bs) ++kd;
    else { ++ks; ++kd; }
  }
  return cnt;
}

__device__ void lpt_assign(const PlanArgs& a, int l, uint64_t* keys) {
  const int tid = threadIdx.x;
  const int64_t N = a.N;
  const int D = a.lay[l].dp;
  int64_t n2 = 1;
  while (n2 < N) n2 <<= 1;
  // key: (L desc, i asc) == ascending (INT32_MAX - L, i)
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
  // Graham's greedy: least-loaded group, ties to the lowest index.  One thread; the D <= 8
  // loads live in registers and L is recovered from the sort key (no dependent global load).
  if (tid == 0) {
    int64_t ld[kMaxShards];
#pragma unroll
    for (int g = 0; g < kMaxShards; ++g) ld[g] = 0;
    for (int64_t q = 0; q < N; ++q) {
      const uint64_t key = keys[q];
      const int i = (int)(key & 0xffffffffu);
      const int64_t L = (int64_t)(0x7fffffffu - (uint32_t)(key >> 32));
      int best = 0;
      int64_t bl = ld[0];
#pragma unroll
      for (int g = 1; g < kMaxShards; ++g)
        if (g < D && ld[g] < bl) { bl = ld[g]; best = g; }
#pragma unroll
      for (int g = 0; g < kMaxShards; ++g)
        if (g == best) ld[g] += L;
      a.grp[l][i] = best;
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(NT, 1) planner_kernel(const PlanArgs a) {
  extern __shared__ uint64_t lpt_keys[];
  __shared__ int64_t sm_scan[NT / 32 + 1];
  __shared__ PartitionSmem ps;
  PlanHeader* h = a.hdr;
  const int tid = threadIdx.x;
  const int64_t N = a.N;

  // ---- phase 0: lengths, P, T -------------------------------------------------------
  const int64_t T = tile_scan(
      N,
      [&](int64_t i) {
        int32_t L = a.seq_lens[i];
        if (L < 0) { latch(h, EARL_ERR_INVALID_ARGUMENT, (int)i); L = 0; }
        a.lens[i] = L;
        return (int64_t)L;
      },
      [&](int64_t i, int64_t ex) { a.P[i] = ex; }, sm_scan);
  if (tid == 0) { a.P[N] = T; h->T = T; }
  __syncthreads();

  // ---- phase 1: assignment -----------------------------------------------------------
  for (int l = 0; l < 2; ++l) {
    const LayoutDesc& L = a.lay[l];
    const int D = L.dp;
    if (L.assign == EARL_ASSIGN_LPT) {
      lpt_assign(a, l, lpt_keys);
      continue;
    }
    for (int64_t i = tid; i < N; i += NT) {
      int g = 0;
      if (L.assign == EARL_ASSIGN_GIVEN_COUNTS) {
        while (g < D - 1 && i >= L.count_start[g + 1]) ++g;
      } else if (L.assign == EARL_ASSIGN_CONTIG) {
        if (T == 0) {  // count blocks, earlier groups take the extra
          const int64_t q = N / D, r = N % D;
          g = (i < r * (q + 1)) ? (int)(i / (q + 1)) : (int)(r + (i - r * (q + 1)) / q);
        } else {
          const int64_t m = ((int64_t)D * (2 * a.P[i] + a.lens[i])) / (2 * T);
          g = (int)(m < D - 1 ? m : D - 1);
        }
      } else {  // EXPLICIT
        g = L.group_of_seq[i];
        if (g < 0 || g >= D) { latch(h, EARL_ERR_LAYOUT, (int)i); g = 0; }
      }
      a.grp[l][i] = g;
    }
  }
  __syncthreads();

  // ---- phase 2: per-layout group order and local token offsets ------------------------
  for (int l = 0; l < 2; ++l) {
    const LayoutDesc& L = a.lay[l];
    const int D = L.dp, SP = L.sp;
    int32_t* grp = a.grp[l];
    int32_t* perm = a.perm[l];
    stable_partition(
        N, D, [&](int64_t i) { return grp[i]; },
        [&](int64_t i, int64_t pos) { perm[pos] = (int32_t)i; }, ps);
    if (tid <= D) h->group_start[l][tid] = ps.bstart[tid];
    if (tid < D) h->group_count[l][tid] = ps.bstart[tid + 1] - ps.bstart[tid];
    __syncthreads();
    for (int k = 0; k < SP; ++k) {
      int64_t* cum = a.cum[l] + (int64_t)k * (N + 1);
      int64_t* off = a.off[l] + (int64_t)k * N;
      const int64_t tot = tile_scan(
          N, [&](int64_t j) { return chunk_len(a.lens[perm[j]], SP, k); },
          [&](int64_t j, int64_t ex) { cum[j] = ex; }, sm_scan);
      if (tid == 0) cum[N] = tot;
      __syncthreads();
      for (int64_t j = tid; j < N; j += NT) {
        const int i = perm[j];
        off[i] = cum[j] - cum[h->group_start[l][grp[i]]];
      }
      if (tid < D) {
        const int64_t st = cum[h->group_start[l][tid + 1]] - cum[h->group_start[l][tid]];
        h->shard_tokens[l][tid * SP + k] = st;
        if (l == 1 && st > 0x7fffffffLL) latch(h, EARL_ERR_CAPACITY, tid * SP + k);
      }
      __syncthreads();
    }
  }

  // ---- phase 3: pieces ----------------------------------------------------------------
  const LayoutDesc& S = a.lay[0];
  const LayoutDesc& Dl = a.lay[1];
  const int Sd = Dl.dp * Dl.sp;
  const int64_t M = tile_scan(
      N,
      [&](int64_t i) {
        return (int64_t)for_each_piece(a.lens[i], S.sp, Dl.sp, [](int, int, int64_t, int64_t) {});
      },
      [&](int64_t i, int64_t ex) { a.pbase[i] = ex; }, sm_scan);
  if (tid == 0) { a.pbase[N] = M; h->n_pieces = M; }
  __syncthreads();
  for (int64_t i = tid; i < N; i += NT) {
    int64_t p = a.pbase[i];
    const int ss0 = a.grp[0][i] * S.sp, ds0 = a.grp[1][i] * Dl.sp;
    for_each_piece(a.lens[i], S.sp, Dl.sp, [&](int ks, int kd, int64_t x, int64_t y) {
      a.pc_i[p] = (int32_t)i;
      a.pc_x[p] = (int32_t)x;
      a.pc_y[p] = (int32_t)y;
      a.pc_kk[p] = ks | (kd << 8) | (((ss0 + ks) * Sd + ds0 + kd) << 16);
      ++p;
    });
  }
  __syncthreads();

  // ---- phase 4: pieces by message key, message token offsets -------------------------
  const int K = S.dp * S.sp * Sd;
  stable_partition(
      M, K, [&](int64_t q) { return a.pc_kk[q] >> 16; },
      [&](int64_t q, int64_t pos) {
        a.ps_i[pos] = a.pc_i[q];
        a.ps_x[pos] = a.pc_x[q];
        a.ps_y[pos] = a.pc_y[q];
        a.ps_kk[pos] = a.pc_kk[q];
      },
      ps);
  if (tid <= K) h->key_piece_start[tid] = ps.bstart[tid];
  if (tid < K) h->key_pieces[tid] = ps.bstart[tid + 1] - ps.bstart[tid];
  __syncthreads();
  const int64_t Mtok = tile_scan(
      M, [&](int64_t q) { return (int64_t)(a.ps_y[q] - a.ps_x[q]); },
      [&](int64_t q, int64_t ex) { a.ps_scan[q] = ex; }, sm_scan);
  if (tid == 0) a.ps_scan[M] = Mtok;
  __syncthreads();
  if (tid < K)
    h->key_tokens[tid] = a.ps_scan[h->key_piece_start[tid + 1]] - a.ps_scan[h->key_piece_start[tid]];
  __syncthreads();

  // ---- phase 5: bases and message offsets (one thread; <= 8 x 8 entries) --------------
  const int nts = S.tp < Dl.tp ? S.tp : Dl.tp;
  if (tid == 0) {
    int64_t rec = 0, tok = 0;
    for (int r = 0; r < a.world; ++r) {
      h->rec_begin[r] = rec;
      h->rec_tok_begin[r] = tok;
      const int rr = r - S.rank0;
      const bool in_src = rr >= 0 && rr < S.dp * S.sp * S.tp;
      const int ss = in_src ? rr / S.tp : 0, ts = in_src ? rr % S.tp : 0;
      for (int ds = 0; ds < Sd; ++ds) {
        h->rec_base[r][ds] = rec;
        h->rec_tok_base[r][ds] = tok;
        if (in_src && ts < nts) {
          rec += h->key_pieces[ss * Sd + ds];
          tok += h->key_tokens[ss * Sd + ds];
        }
      }
    }
    h->rec_begin[a.world] = rec;
    h->rec_tok_begin[a.world] = tok;
    h->n_records = rec;
    h->rec_tokens = tok;
    for (int ss = 0; ss < S.dp * S.sp; ++ss) {
      int64_t off = 0;
      for (int ds = 0; ds < Sd; ++ds) {
        h->msg_off[ss * Sd + ds] = off;
        for (int f = 0; f < a.n_fields; ++f)
          off += (h->key_tokens[ss * Sd + ds] * a.Bf[f] + 15) & ~15LL;
      }
      h->stage_bytes_shard[ss] = off;
    }
    a.rec.tok_prefix[rec] = tok;
  }
  __syncthreads();

  // ---- phase 6: records ---------------------------------------------------------------
  const int64_t nrec = M * nts;
  for (int64_t idx = tid; idx < nrec; idx += NT) {
    const int64_t q = idx / nts;
    const int ts = (int)(idx - q * nts);
    const int kk = a.ps_kk[q];
    const int ks = kk & 0xff, kd = (kk >> 8) & 0xff, key = kk >> 16;
    const int ss = key / Sd, ds = key - ss * Sd;
    const int s = S.rank0 + ss * S.tp + ts;
    const int64_t rho = q - h->key_piece_start[key];
    const int64_t j = h->rec_base[s][ds] + rho;
    const int i = a.ps_i[q];
    const int64_t x = a.ps_x[q], y = a.ps_y[q];
    const int64_t L = a.lens[i];
    const int64_t msg_tok = a.ps_scan[q] - a.ps_scan[h->key_piece_start[key]];
    a.rec.seq[j] = i;
    a.rec.x[j] = (int32_t)x;
    a.rec.n[j] = (int32_t)(y - x);
    a.rec.code[j] = (uint32_t)s | ((uint32_t)ss << 8) | ((uint32_t)ds << 16) | ((uint32_t)ts << 24);
    a.rec.src_tok[j] = a.off[0][(int64_t)ks * N + i] + (x - chunk_lo(L, S.sp, ks));
    a.rec.dst_tok[j] = a.off[1][(int64_t)kd * N + i] + (x - chunk_lo(L, Dl.sp, kd));
    a.rec.msg_tok[j] = msg_tok;
    a.rec.tok_prefix[j] = h->rec_tok_base[s][ds] + msg_tok;
  }
}

// Destination metadata of dst shard (g, k): cu_seqlens (int32), seq_ids (int64), tok_start.
__global__ void local_meta_kernel(const PlanArgs a, int g, int k, int32_t* cu, int64_t* ids,
                                  int32_t* tok_start) {
  const PlanHeader* h = a.hdr;
  const int64_t N = a.N;
  const int64_t n = h->group_count[1][g];
  const int64_t gs = h->group_start[1][g];
  const int64_t* cum = a.cum[1] + (int64_t)k * (N + 1);
  const int sp = a.lay[1].sp;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j <= n;
       j += (int64_t)gridDim.x * blockDim.x) {
    if (cu) cu[j] = (int32_t)(cum[gs + j] - cum[gs]);
    if (j < n) {
      const int i = a.perm[1][gs + j];
      if (ids) ids[j] = i;
      if (tok_start) tok_start[j] = (int32_t)chunk_lo(a.lens[i], sp, k);
    }
  }
}

}  // namespace

cudaError_t launch_planner(const PlanArgs& a, size_t lpt_smem, cudaStream_t s) {
  if (lpt_smem > 0) {
    cudaError_t e = cudaFuncSetAttribute(planner_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)lpt_smem);
    if (e != cudaSuccess) return e;
  }
  planner_kernel<<<1, NT, lpt_smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_local_meta(const PlanArgs& a, int g, int k, int32_t* cu, int64_t* ids,
                              int32_t* tok_start, cudaStream_t s) {
  local_meta_kernel<<<64, 256, 0, s>>>(a, g, k, cu, ids, tok_start);
  return cudaGetLastError();
}

}  // namespace earl
