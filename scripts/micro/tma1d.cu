// Microbenchmark: moving misaligned 4-B-field pieces (source and destination token offsets not
// congruent mod 16 B) by 1-D tensor TMA (cp.async.bulk.tensor with element coordinates) against
// the same bytes as contiguous aligned pieces.  Probe for the copy engine's realign path
// (DESIGN.md §10 next, item 2).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o
// tma1d tma1d.cu -lcuda ; run: ./tma1d
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int kBox = 256;          // elements per tensor op (fp32: 1 KB)
constexpr int kWarps = 8;
constexpr int kStages = 3;
constexpr int kStageBoxes = 8;     // 8 KB stages
constexpr int kStageBytes = kBox * 4 * kStageBoxes;

struct Piece { int64_t s, d, n; };  // element offsets and count (n multiple of kBox here)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(kWarps * 32, 1) tma_copy(const __grid_constant__ CUtensorMap src,
                                                        const __grid_constant__ CUtensorMap dst,
                                                        const Piece* pieces, int np, unsigned* ctr) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[kWarps][kStages];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint8_t* ring = sm + (size_t)w * kStages * kStageBytes;
  if (lane == 0) {
    for (int s = 0; s < kStages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[w][s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  if (lane != 0) return;  // one thread drives the warp's ring
  // work: stages of up to kStageBoxes boxes, walking claimed pieces
  int pi = -1; int64_t pos = 0;
  auto next_box = [&](int64_t& se, int64_t& de) -> bool {
    while (pi < 0 || pos >= pieces[pi].n) {
      pi = (int)atomicAdd(ctr, 1u);
      if (pi >= np) return false;
      pos = 0;
    }
    se = pieces[pi].s + pos; de = pieces[pi].d + pos; pos += kBox;
    return true;
  };
  int64_t dco[kStages][kStageBoxes];
  int nbx[kStages];
  auto fill = [&](int s) -> bool {
    int n = 0;
    int64_t se, de;
    while (n < kStageBoxes && next_box(se, de)) {
      dco[s][n] = de;
      const uint32_t dstp = smem_u32(ring + (size_t)s * kStageBytes + n * kBox * 4);
      ++n;
      asm volatile("cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];"
                   ::"r"(dstp), "l"(&src), "r"((int)se), "r"(smem_u32(&bar[w][s])) : "memory");
    }
    nbx[s] = n;
    if (n == 0) return false;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[w][s])), "r"(n * kBox * 4) : "memory");
    return true;
  };
  int issued = 0;
  for (int s = 0; s < kStages - 1; ++s) if (fill(s)) ++issued; else break;
  for (int c = 0; c < issued; ++c) {
    const int s = c % kStages;
    uint32_t done = 0;
    const uint32_t par = (uint32_t)((c / kStages) & 1);
    while (!done)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done) : "r"(smem_u32(&bar[w][s])), "r"(par) : "memory");
    for (int k = 0; k < nbx[s]; ++k)
      asm volatile("cp.async.bulk.tensor.1d.global.shared::cta.bulk_group [%0, {%1}], [%2];"
                   ::"l"(&dst), "r"((int)dco[s][k]), "r"(smem_u32(ring + (size_t)s * kStageBytes + k * kBox * 4)) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    const int ns = (c + kStages - 1) % kStages;
    if (fill(ns)) ++issued;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void init(float* a, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = (float)(i & 0xffffff);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int64_t N = int64_t(1) << 30;  // 1 Gi fp32 elements = 4 GiB per buffer
  float *a, *b;
  CK(cudaMalloc(&a, N * 4));
  CK(cudaMalloc(&b, N * 4));
  init<<<1184, 256>>>(a, N);
  CK(cudaDeviceSynchronize());
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  EncodeFn enc = (EncodeFn)fn;
  CUtensorMap ms, md;
  cuuint64_t dims[1] = {(cuuint64_t)N}, strides[1] = {(cuuint64_t)N * 4};
  cuuint32_t box[1] = {kBox}, es[1] = {1};
  if (enc(&ms, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 1, a, dims, strides + 0, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
      enc(&md, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 1, b, dims, strides + 0, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n");
    return 1;
  }
  // pieces: lengths ~ multiples of kBox (2048 +- ...), source contiguous from offset 1, destination
  // contiguous from offset 3 with a shuffled order: never congruent mod 4 elements
  std::mt19937_64 rng(1);
  for (int mode = 0; mode < 2; ++mode) {
    std::vector<Piece> ps;
    int64_t so = mode ? 1 : 0, total = 0;
    while (so + 8192 < N - 8192) {
      const int64_t n = kBox * (1 + (int64_t)(rng() % 16));
      ps.push_back({so, 0, n});
      so += n + (mode ? (int64_t)(rng() % 3) + 1 : 0);
      total += n;
    }
    std::vector<int> order(ps.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
    std::shuffle(order.begin(), order.end(), rng);
    int64_t dpos = mode ? 3 : 0;
    for (int i : order) { ps[i].d = dpos; dpos += ps[i].n + (mode ? (int64_t)(rng() % 3) + 1 : 0); }
    Piece* dp;
    unsigned* ctr;
    CK(cudaMalloc(&dp, ps.size() * sizeof(Piece)));
    CK(cudaMalloc(&ctr, 4));
    CK(cudaMemcpy(dp, ps.data(), ps.size() * sizeof(Piece), cudaMemcpyHostToDevice));
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t smem = (size_t)kWarps * kStages * kStageBytes;
    CK(cudaFuncSetAttribute(tma_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int it = 0; it < 6; ++it) {
      CK(cudaMemset(ctr, 0, 4));
      cudaEventRecord(e0);
      tma_copy<<<sms, kWarps * 32, smem>>>(ms, md, dp, (int)ps.size(), ctr);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms_ = 0;
      cudaEventElapsedTime(&ms_, e0, e1);
      if (it > 0) best = std::min(best, ms_);
    }
    CK(cudaGetLastError());
    int bad = 0;
    for (int k = 0; k < 5; ++k) {
      const Piece& P = ps[(rng() % ps.size())];
      std::vector<float> x(P.n), y(P.n);
      CK(cudaMemcpy(x.data(), a + P.s, P.n * 4, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(y.data(), b + P.d, P.n * 4, cudaMemcpyDeviceToHost));
      for (int64_t i = 0; i < P.n; ++i) bad += x[i] != y[i];
    }
    printf("check: %s; ", bad ? "MISMATCH" : "ok");
    printf("%s pieces=%zu elements=%lld: %.3f ms, %.1f GB/s (read+write)\n", mode ? "misaligned" : "aligned   ",
           ps.size(), (long long)total, best, 2.0 * total * 4 / (best * 1e-3) / 1e9);
    cudaFree(dp); cudaFree(ctr);
  }
  return 0;
}
