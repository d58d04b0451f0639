/* abi_smoke.c -- the C ABI used from plain C (no Python, no torch).
 *
 *   ./abi_smoke          : no GPU needed; version, status strings, argument validation
 *   ./abi_smoke gpu      : emulated 2-rank comm on device 0: BASELINE configs[0] (8 sequences
 *                          L = [5,17,64,9,33,12,48,21], src DP2 GIVEN_COUNTS [4,4] -> dst DP1),
 *                          one int32 field whose token t of sequence i holds 1000*i + t; checks
 *                          the destination bytes, cu_seqlens and the plan export against the
 *                          hand-worked values of tests/golden/c1_tiny.json; then the device
 *                          length gather, a per-sequence field plan and option validation.
 * Exit code 0 on success.
 */
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "earl_dispatch.h"

#define CHECK(cond, ...)                         \
  do {                                           \
    if (!(cond)) {                               \
      fprintf(stderr, "FAIL %s:%d: ", __FILE__, __LINE__); \
      fprintf(stderr, __VA_ARGS__);              \
      fprintf(stderr, "\n");                     \
      return 1;                                  \
    }                                            \
  } while (0)

static int no_gpu_part(void) {
  earl_comm_t c = NULL;
  CHECK(earl_abi_version() == EARL_ABI_VERSION, "abi version");
  CHECK(strcmp(earl_status_string(EARL_ERR_LAYOUT), "EARL_ERR_LAYOUT") == 0, "status string");
  CHECK(earl_comm_create(0, 9, 0, 0, &c) == EARL_ERR_UNSUPPORTED, "world 9 must be unsupported");
  CHECK(strstr(earl_last_error(), "world 9") != NULL, "last error names the world: %s", earl_last_error());
  CHECK(earl_comm_create(3, 2, 0, 0, &c) == EARL_ERR_INVALID_ARGUMENT, "rank 3 of 2");
  CHECK(earl_comm_create(0, 2, 0, 0, NULL) == EARL_ERR_INVALID_ARGUMENT, "NULL out");
  CHECK(earl_dispatch_plan(NULL, NULL, NULL, NULL, 0, NULL, 0, NULL, NULL) == EARL_ERR_INVALID_ARGUMENT, "NULL plan args");
  CHECK(earl_comm_destroy(NULL) == EARL_OK && earl_plan_destroy(NULL) == EARL_OK, "destroy NULL");
  printf("abi_smoke: no-GPU checks passed\n");
  return 0;
}

static int gpu_part(void) {
  const int32_t L[8] = {5, 17, 64, 9, 33, 12, 48, 21};
  const int64_t counts[2] = {4, 4};
  int32_t host_src[2][128];
  int32_t want[209];
  int n_tok[2] = {0, 0};
  int k = 0;
  for (int i = 0; i < 8; ++i)
    for (int t = 0; t < L[i]; ++t) {
      host_src[i / 4][n_tok[i / 4]++] = 1000 * i + t;
      want[k++] = 1000 * i + t;
    }
  CHECK(n_tok[0] == 95 && n_tok[1] == 114 && k == 209, "token counts");

  earl_comm_t comm = NULL;
  CHECK(earl_comm_create(EARL_ALL_RANKS, 2, 0, 0, &comm) == EARL_OK, "comm: %s", earl_last_error());
  int32_t* d_lens = NULL;
  void* d_src[2] = {NULL, NULL};
  void* d_dst[2] = {NULL, NULL};
  CHECK(cudaMalloc((void**)&d_lens, sizeof(L)) == cudaSuccess, "malloc");
  CHECK(cudaMemcpy(d_lens, L, sizeof(L), cudaMemcpyHostToDevice) == cudaSuccess, "copy");
  for (int r = 0; r < 2; ++r) {
    CHECK(cudaMalloc(&d_src[r], 128 * 4) == cudaSuccess, "malloc");
    CHECK(cudaMemcpy(d_src[r], host_src[r], n_tok[r] * 4, cudaMemcpyHostToDevice) == cudaSuccess, "copy");
  }
  earl_layout_t src = {0, 2, 1, 1, EARL_ASSIGN_GIVEN_COUNTS, EARL_SP_BLOCK, 0, 0, counts, NULL};
  earl_layout_t dst = {0, 1, 1, 1, EARL_ASSIGN_CONTIG, EARL_SP_BLOCK, 0, 0, NULL, NULL};
  earl_field_t field = {4, 1};
  earl_plan_t plan = NULL;
  CHECK(earl_dispatch_plan(comm, &src, &dst, d_lens, 8, &field, 1, NULL, &plan) == EARL_OK,
        "plan: %s", earl_last_error());
  int64_t ns = 0, nt = 0;
  CHECK(earl_plan_local_sizes(plan, 0, &ns, &nt) == EARL_OK && ns == 8 && nt == 209, "sizes %lld %lld",
        (long long)ns, (long long)nt);
  CHECK(cudaMalloc(&d_dst[0], 209 * 4) == cudaSuccess, "malloc");
  const void* send[2] = {d_src[0], d_src[1]};
  void* recv[2] = {d_dst[0], NULL};
  CHECK(earl_dispatch_exec(plan, send, recv, NULL) == EARL_OK, "exec: %s", earl_last_error());
  int32_t got[209];
  CHECK(cudaMemcpy(got, d_dst[0], sizeof(got), cudaMemcpyDeviceToHost) == cudaSuccess, "copy back");
  CHECK(memcmp(got, want, sizeof(got)) == 0, "destination bytes differ");
  /* per-source dispatch: source ranks 1 then 0 into a cleared buffer give the same bytes */
  CHECK(cudaMemset(d_dst[0], 0, 209 * 4) == cudaSuccess, "memset");
  CHECK(earl_dispatch_exec_src(plan, 1, send, recv, NULL) == EARL_OK, "exec_src 1: %s", earl_last_error());
  CHECK(earl_dispatch_exec_src(plan, 0, send, recv, NULL) == EARL_OK, "exec_src 0: %s", earl_last_error());
  CHECK(earl_dispatch_exec_src(plan, 2, send, recv, NULL) == EARL_ERR_INVALID_ARGUMENT, "exec_src range");
  CHECK(cudaMemcpy(got, d_dst[0], sizeof(got), cudaMemcpyDeviceToHost) == cudaSuccess, "copy back");
  CHECK(memcmp(got, want, sizeof(got)) == 0, "per-source destination bytes differ");
  int32_t* d_cu = NULL;
  CHECK(cudaMalloc((void**)&d_cu, 9 * 4) == cudaSuccess, "malloc");
  CHECK(earl_plan_local_meta(plan, 0, d_cu, NULL, NULL, NULL) == EARL_OK, "meta");
  int32_t cu[9];
  CHECK(cudaMemcpy(cu, d_cu, sizeof(cu), cudaMemcpyDeviceToHost) == cudaSuccess, "copy back");
  const int32_t want_cu[9] = {0, 5, 22, 86, 95, 128, 140, 188, 209};  /* golden c1 dp2_to_dp1 */
  CHECK(memcmp(cu, want_cu, sizeof(cu)) == 0, "cu_seqlens differ");
  earl_plan_stats_t st;
  CHECK(earl_plan_stats(plan, &st) == EARL_OK, "stats");
  CHECK(st.moved_bytes == 456 && st.total_bytes == 836, "moved %llu total %llu",
        (unsigned long long)st.moved_bytes, (unsigned long long)st.total_bytes);
  int64_t nseg = 0;
  CHECK(earl_plan_export(plan, 0, &nseg, NULL, NULL, NULL, NULL, NULL, NULL, NULL) == EARL_OK && nseg == 8, "export count");
  int32_t s[8], d[8], x[8], y[8];
  int64_t seq[8], so[8], dof[8];
  CHECK(earl_plan_export(plan, 8, &nseg, s, d, seq, x, y, so, dof) == EARL_OK, "export");
  for (int j = 0; j < 8; ++j) {
    CHECK(seq[j] == j && s[j] == (j < 4 ? 0 : 1) && d[j] == 0 && x[j] == 0 && y[j] == L[j], "segment %d", j);
    CHECK(dof[j] == want_cu[j], "segment %d dst offset", j);
  }
  /* step a1 on the device: the two ranks' local lengths, gathered rank-major */
  int32_t* d_loc[2] = {NULL, NULL};
  int32_t* d_glob = NULL;
  for (int r = 0; r < 2; ++r) {
    CHECK(cudaMalloc((void**)&d_loc[r], 4 * 4) == cudaSuccess, "malloc");
    CHECK(cudaMemcpy(d_loc[r], L + 4 * r, 4 * 4, cudaMemcpyHostToDevice) == cudaSuccess, "copy");
  }
  CHECK(cudaMalloc((void**)&d_glob, sizeof(L)) == cudaSuccess, "malloc");
  const void* loc[2] = {d_loc[0], d_loc[1]};
  CHECK(earl_allgather_lengths(comm, counts, loc, d_glob, NULL) == EARL_OK, "gather: %s", earl_last_error());
  int32_t glob[8];
  CHECK(cudaMemcpy(glob, d_glob, sizeof(glob), cudaMemcpyDeviceToHost) == cudaSuccess, "copy back");
  CHECK(memcmp(glob, L, sizeof(L)) == 0, "gathered lengths differ");
  /* per-sequence fields (reading n4): one int32 record per sequence, routed with the token plan */
  earl_plan_t splan = NULL;
  earl_field_t rec = {4, 1};
  CHECK(earl_plan_seq_fields(plan, &rec, 1, NULL, &splan) == EARL_OK, "seq plan: %s", earl_last_error());
  int32_t host_rec[2][4];
  for (int i = 0; i < 8; ++i) host_rec[i / 4][i % 4] = 7 * i + 1;
  void* d_rec_src[2] = {NULL, NULL};
  void* d_rec_dst = NULL;
  for (int r = 0; r < 2; ++r) {
    CHECK(cudaMalloc(&d_rec_src[r], 16) == cudaSuccess, "malloc");
    CHECK(cudaMemcpy(d_rec_src[r], host_rec[r], 16, cudaMemcpyHostToDevice) == cudaSuccess, "copy");
  }
  CHECK(cudaMalloc(&d_rec_dst, 32) == cudaSuccess, "malloc");
  const void* rsend[2] = {d_rec_src[0], d_rec_src[1]};
  void* rrecv[2] = {d_rec_dst, NULL};
  CHECK(earl_dispatch_exec(splan, rsend, rrecv, NULL) == EARL_OK, "seq exec: %s", earl_last_error());
  int32_t got_rec[8];
  CHECK(cudaMemcpy(got_rec, d_rec_dst, 32, cudaMemcpyDeviceToHost) == cudaSuccess, "copy back");
  for (int i = 0; i < 8; ++i) CHECK(got_rec[i] == 7 * i + 1, "sequence record %d", i);
  /* options of a multi-process comm are refused on an emulated one, or validated */
  CHECK(earl_comm_set_nodes(comm, 1) == EARL_ERR_UNSUPPORTED, "set_nodes on an emulated comm");
  CHECK(earl_comm_set_exec_options(comm, 2, -1) == EARL_ERR_INVALID_ARGUMENT, "remote_store 2");
  CHECK(earl_comm_set_exec_options(comm, 1, 9) == EARL_ERR_INVALID_ARGUMENT, "shape 9");
  CHECK(earl_comm_set_exec_options(comm, -1, -1) == EARL_OK, "default options");
  earl_plan_destroy(plan);   /* the sequence plan keeps its token plan alive */
  CHECK(earl_dispatch_exec(splan, rsend, rrecv, NULL) == EARL_OK, "seq exec after token destroy");
  CHECK(cudaDeviceSynchronize() == cudaSuccess, "sync");
  earl_plan_destroy(splan);
  earl_comm_destroy(comm);
  cudaFree(d_lens); cudaFree(d_src[0]); cudaFree(d_src[1]); cudaFree(d_dst[0]); cudaFree(d_cu);
  cudaFree(d_loc[0]); cudaFree(d_loc[1]); cudaFree(d_glob); cudaFree(d_rec_src[0]);
  cudaFree(d_rec_src[1]); cudaFree(d_rec_dst);
  printf("abi_smoke: GPU dispatch checks passed\n");
  return 0;
}

int main(int argc, char** argv) {
  if (no_gpu_part()) return 1;
  if (argc > 1 && strcmp(argv[1], "gpu") == 0) return gpu_part();
  return 0;
}
