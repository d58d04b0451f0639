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
#include "earl_internal.cuh"

namespace earl {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kTokPerLane = 8;
constexpr int kTile = 32 * kTokPerLane;

// Source ranks of the launch, each with its sequence count and the start of its sequences in
// the group order (SP = 1: rank = rank0 + g*TP + t, group g).
struct RankTable {
  int n;
  int rank[kMaxWorld];
  int g[kMaxWorld];
  int t[kMaxWorld];
  int64_t count[kMaxWorld];   // sequences of the rank
  int64_t start[kMaxWorld];   // first work item of the rank
  int64_t gstart[kMaxWorld];  // first position of group g in the sorted order
};

__device__ void rank_table(const AggArgs& a, RankTable& rt) {
  const PlanHeader* h = a.hdr;
  const LayoutDesc& S = a.plan.lay[0];
  rt.n = 0;
  int64_t acc = 0;
  for (int r = 0; r < a.world; ++r) {
    if (a.view_rank >= 0 && r != a.view_rank) continue;
    const int q = r - S.rank0;
    if (q < 0 || q >= S.dp * S.tp) continue;
    const int g = q / S.tp, t = q % S.tp;
    rt.rank[rt.n] = r;
    rt.g[rt.n] = g;
    rt.t[rt.n] = t;
    rt.count[rt.n] = h->group_count[0][g];
    rt.gstart[rt.n] = h->group_start[0][g];
    rt.start[rt.n] = acc;
    acc += rt.count[rt.n];
    ++rt.n;
  }
}

// One warp per (rank, sequence) work item; the sequence is walked backwards in tiles of 256
// tokens: every lane reduces its 8 tokens to the affine map x -> S + gamma^8 x, a warp suffix
// scan composes the maps of the lanes to its right, then each lane emits its 8 returns.
__global__ void __launch_bounds__(256) returns_kernel(const __grid_constant__ AggArgs a) {
  __shared__ RankTable rt;
  if (threadIdx.x == 0) rank_table(a, rt);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t total = rt.n ? rt.start[rt.n - 1] + rt.count[rt.n - 1] : 0;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const float gamma = a.gamma;
  double s_m = 0.0, s_g = 0.0, s_g2 = 0.0;
  for (int64_t item = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); item < total;
       item += nwarps) {
    int ri = 0;
    while (ri + 1 < rt.n && item >= rt.start[ri + 1]) ++ri;
    const int r = rt.rank[ri];
    const int64_t pos = rt.gstart[ri] + (item - rt.start[ri]);
    const int i = a.plan.perm[0][pos];
    const int64_t L = a.plan.lens[i];
    const int64_t o = a.plan.off[0][i];  // SP = 1: chunk 0 is the whole sequence
    const float* rw = a.rewards[r] + o;
    const uint8_t* mk = a.mask[r] + o;
    float* G = a.returns[r] + o;
    const bool count_stats = rt.t[ri] == 0;
    float carry = 0.f;  // G of the first token right of the current tile
    for (int64_t tile_end = L; tile_end > 0; tile_end -= kTile) {
      const int64_t tile_beg = tile_end > kTile ? tile_end - kTile : 0;
      const int64_t t0 = tile_beg + (int64_t)lane * kTokPerLane;
      float v[kTokPerLane];
#pragma unroll
      for (int k = 0; k < kTokPerLane; ++k) {
        const int64_t tt = t0 + k;
        v[k] = (tt < tile_end) ? rw[tt] * (float)mk[tt] : 0.f;
      }
      // lane's own map: S = sum_k gamma^k v[k] (over its valid tokens), P = gamma^(#valid)
      float S = 0.f, P = 1.f;
#pragma unroll
      for (int k = kTokPerLane - 1; k >= 0; --k) {
        if (t0 + k < tile_end) { S = v[k] + gamma * S; P *= gamma; }
      }
      // suffix composition over lanes > lane: (S1,P1) o (S2,P2) = (S1 + P1 S2, P1 P2)
      float sS = S, sP = P;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const float oS = __shfl_down_sync(kFull, sS, off), oP = __shfl_down_sync(kFull, sP, off);
        if (lane + off < 32) { sS = sS + sP * oS; sP = sP * oP; }
      }
      // exclusive suffix: the map of lanes right of this one, applied to the tile's carry
      float rS = __shfl_down_sync(kFull, sS, 1), rP = __shfl_down_sync(kFull, sP, 1);
      if (lane == 31) { rS = 0.f; rP = 1.f; }
      float g_next = rS + rP * carry;
#pragma unroll
      for (int k = kTokPerLane - 1; k >= 0; --k) {
        const int64_t tt = t0 + k;
        if (tt < tile_end) {
          const float gk = v[k] + gamma * g_next;
          G[tt] = gk;
          if (count_stats && mk[tt]) {
            s_m += 1.0;
            s_g += (double)gk;
            s_g2 += (double)gk * (double)gk;
          }
          g_next = gk;
        }
      }
      carry = __shfl_sync(kFull, sS + sP * carry, 0);
    }
    if (lane == 0 && a.seq_return != nullptr && a.seq_return[r] != nullptr)
      a.seq_return[r][item - rt.start[ri]] = (L > 0) ? G[0] : 0.f;
  }
  // warp, then block reduction of the fp64 partials; one atomic per block
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    s_m += __shfl_xor_sync(kFull, s_m, off);
    s_g += __shfl_xor_sync(kFull, s_g, off);
    s_g2 += __shfl_xor_sync(kFull, s_g2, off);
  }
  __shared__ double red[3][8];
  const int w = threadIdx.x >> 5;
  if (lane == 0) { red[0][w] = s_m; red[1][w] = s_g; red[2][w] = s_g2; }
  __syncthreads();
  if (threadIdx.x < 3) {
    double acc = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) acc += red[threadIdx.x][k];
    if (acc != 0.0) atomicAdd(a.partial + threadIdx.x, acc);
  }
}

// A_t = m_t (G_t - mu) / (sigma + eps) over every token of the launch's source ranks.
__global__ void __launch_bounds__(256) advantage_kernel(const __grid_constant__ AggArgs a) {
  __shared__ RankTable rt;
  __shared__ float s_mu, s_inv;
  if (threadIdx.x == 0) {
    rank_table(a, rt);
    const double n = a.stats[0];
    const double mu = n > 0 ? a.stats[1] / n : 0.0;
    double var = n > 0 ? a.stats[2] / n - mu * mu : 0.0;
    if (var < 0) var = 0;
    s_mu = (float)mu;
    s_inv = (float)(1.0 / (sqrt(var) + (double)a.eps));
  }
  __syncthreads();
  const float mu = s_mu, inv = s_inv;
  for (int ri = 0; ri < rt.n; ++ri) {
    const int r = rt.rank[ri];
    const int64_t ntok = a.hdr->shard_tokens[0][rt.g[ri]];
    const float* G = a.returns[r];
    const uint8_t* mk = a.mask[r];
    float* A = a.adv[r];
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntok;
         t += (int64_t)gridDim.x * blockDim.x)
      A[t] = mk[t] ? (G[t] - mu) * inv : 0.f;
  }
}

}  // namespace

cudaError_t launch_returns(const AggArgs& a, int sm_count, cudaStream_t s) {
  returns_kernel<<<sm_count * 4, 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_advantages(const AggArgs& a, int sm_count, cudaStream_t s) {
  advantage_kernel<<<sm_count * 8, 256, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace earl
