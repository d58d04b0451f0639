// HBM ceiling for the exec kernel's traffic mix: read one buffer, write it to 4 destinations
// (1R:4W, the TP4-replicated dispatch), next to 1R:1W copy and write-only.  Plain LD/ST
// streaming kernels, grid-stride, CUDA events, best of 10.  Diagnostic only (not the product).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_1r4w(const uint4* __restrict__ s, uint4* __restrict__ d0, uint4* __restrict__ d1,
                       uint4* __restrict__ d2, uint4* __restrict__ d3, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const uint4 v = __ldcs(s + i);
    __stcs(d0 + i, v); __stcs(d1 + i, v); __stcs(d2 + i, v); __stcs(d3 + i, v);
  }
}
__global__ void k_1r1w(const uint4* __restrict__ s, uint4* __restrict__ d0, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(d0 + i, __ldcs(s + i));
}
__global__ void k_w(uint4* __restrict__ d0, size_t n) {
  const uint4 v = make_uint4(1, 2, 3, 4);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(d0 + i, v);
}

template <class F>
float best(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float m = 1e9f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < m) m = ms;
  }
  return m;
}

int main() {
  const size_t bytes = 1ull << 30, n = bytes / 16;
  uint4 *s, *d[4];
  cudaMalloc(&s, bytes); cudaMemset(s, 1, bytes);
  for (auto& p : d) { cudaMalloc(&p, bytes); cudaMemset(p, 0, bytes); }
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int per : {4, 8, 16}) {
    const int grid = sms * per;
    float t4 = best([&] { k_1r4w<<<grid, 256>>>(s, d[0], d[1], d[2], d[3], n); });
    float t1 = best([&] { k_1r1w<<<grid, 256>>>(s, d[0], n); });
    float tw = best([&] { k_w<<<grid, 256>>>(d[0], n); });
    printf("{\"ctas_per_sm\": %d, \"1R4W_GBps\": %.1f, \"1R1W_GBps\": %.1f, \"write_only_GBps\": %.1f}\n", per,
           5.0 * bytes / (t4 * 1e-3) / 1e9, 2.0 * bytes / (t1 * 1e-3) / 1e9, 1.0 * bytes / (tw * 1e-3) / 1e9);
  }
  return 0;
}
