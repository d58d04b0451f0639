// Grid-barrier latency on B200: cooperative_groups grid.sync() against a one-counter
// generation barrier (atom.add.release + ld.acquire spin), 1024-thread CTAs as the planner.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gsync gsync.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ unsigned g_ctr, g_gen;

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ void gen_barrier() {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned gen = ld_acq(&g_gen);
    if (atom_add_acqrel(&g_ctr, 1u) == gridDim.x - 1) {
      g_ctr = 0;
      st_rel(&g_gen, gen + 1);
    } else {
      while (ld_acq(&g_gen) == gen) {}
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(1024, 1) k_cg(int iters, int* out) {
  int acc = 0;
  for (int i = 0; i < iters; ++i) {
    cg::this_grid().sync();
    acc += threadIdx.x;
  }
  if (acc == -1) out[0] = acc;
}
__global__ void __launch_bounds__(1024, 1) k_gen(int iters, int* out) {
  int acc = 0;
  for (int i = 0; i < iters; ++i) {
    gen_barrier();
    acc += threadIdx.x;
  }
  if (acc == -1) out[0] = acc;
}

int main() {
  int* out;
  cudaMalloc(&out, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 200;
  for (int G : {1, 7, 10, 39, 148}) {
    for (int kind = 0; kind < 2; ++kind) {
      void* args[] = {(void*)&iters, (void*)&out};
      void* fn = kind ? (void*)k_gen : (void*)k_cg;
      float best = 1e9f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(a);
        cudaError_t e = cudaLaunchCooperativeKernel(fn, G, 1024, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        if (e != cudaSuccess) { printf("launch failed %s\n", cudaGetErrorString(e)); return 1; }
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("G=%3d %-22s %.2f us per barrier\n", G, kind ? "generation barrier" : "cg grid.sync", best * 1e3f / iters);
    }
  }
  return 0;
}
