// earl_internal.cuh -- device-side data structures shared by the planner, the copy kernels
// and the host glue of libearl_dispatch.so.  (Not part of the C ABI.)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/earl_dispatch.h"

namespace earl {

constexpr int kMaxWorld = EARL_MAX_WORLD;   // 8
constexpr int kMaxFields = EARL_MAX_FIELDS; // 16
constexpr int kMaxShards = 8;               // dp*sp <= world <= 8 per layout
constexpr int kMaxKeys = kMaxShards * kMaxShards;  // (src shard, dst shard) message keys
constexpr int kPlanThreads = 1024;          // the planner is one CTA
constexpr int kPadBytes = 4096;             // signal pad at the start of every window
constexpr int kMaxPlanGrid = 256;           // planner CTAs (cooperative grid) at most

// Layout as the device sees it.  shard = g*sp + k ; rank = rank0 + shard*tp + t.
struct LayoutDesc {
  int32_t rank0, dp, sp, tp, assign;
  int32_t split;            // earl_sp_split_t
  int32_t min_len;          // EARL_SP_THRESHOLD
  int32_t pad_;
  int64_t count_start[kMaxShards + 1];  // GIVEN_COUNTS: prefix of counts
  const int32_t* group_of_seq;          // EXPLICIT
};

// Written by the planner into device memory; read by the copy kernels and (after a sync)
// by the host.  Small fixed-size tables only.
struct PlanHeader {
  int32_t err;          // earl_status_t latched on the device (first error wins)
  int32_t err_detail;   // e.g. peer mask for TIMEOUT, offending index for LAYOUT
  int64_t T;            // total tokens
  int64_t n_pieces;
  int64_t n_records;
  int64_t rec_tokens;   // tokens over all records
  int64_t group_count[2][kMaxShards];
  int64_t group_start[2][kMaxShards + 1];
  int64_t shard_tokens[2][kMaxShards];      // tokens held per shard (g*sp+k) of each layout
  int64_t group_tokens[2][kMaxShards];      // tokens of every DP group (FLAT stream length)
  int64_t key_pieces[kMaxKeys];
  int64_t key_piece_start[kMaxKeys + 1];
  int64_t key_tokens[kMaxKeys];             // tokens of message key (ss, ds)
  int64_t msg_off[kMaxKeys];                // byte offset of message (ss, ds) in a stage buffer
  int64_t stage_bytes_shard[kMaxShards];    // stage buffer size of a rank of src shard ss
  int64_t rec_begin[kMaxWorld + 1];         // records of source comm rank r: [rec_begin[r], rec_begin[r+1])
  int64_t rec_tok_begin[kMaxWorld + 1];     // tokens of those records (prefix)
  int64_t rec_base[kMaxWorld][kMaxShards];  // first record of block (s, ds)
  int64_t rec_tok_base[kMaxWorld][kMaxShards];
  int64_t max_len;      // the batch's longest sequence (returns: unit kernel or windowed)
  uint32_t work_ctr;    // copy kernels: dynamic work-unit counter (reset by the last CTA)
  uint32_t fin_ctr;     // copy kernels: finished-CTA counter
};

// Copy records: one per (piece, sending replica ts < min(tp_src, tp_dst)), ordered by
// (s, ds, i, x).  A record feeds destination replicas td = ts, ts+tp_src, ... < tp_dst.
struct Records {
  int32_t* seq;       // global sequence index i
  int32_t* x;         // first token of the piece inside sequence i
  int32_t* n;         // tokens in the piece (y - x)
  uint32_t* code;     // s | ss<<8 | ds<<16 | ts<<24
  int64_t* src_tok;   // token offset in the source rank's field arrays
  int64_t* dst_tok;   // token offset in each destination replica's field arrays
  int64_t* msg_tok;   // token offset inside message (ss, ds)
  int64_t* tok_prefix;// [n_records + 1]: token prefix over records (= rec_tok_base + msg_tok)
};

struct PlanArgs {
  LayoutDesc lay[2];  // 0 = src, 1 = dst
  int64_t N;
  int32_t world;
  int32_t n_fields;
  uint32_t Bf[kMaxFields];
  const int32_t* seq_lens;   // user's device array
  PlanHeader* hdr;
  // per-sequence scratch
  int32_t* lens;             // [N]
  int64_t* P;                // [N+1]
  int32_t* grp[2];           // [N]
  int32_t* perm[2];          // [N] sorted position -> i
  int64_t* off[2];           // [sp][N] local token offset of chunk k of sequence i
  int64_t* cum[2];           // [sp][N+1] scan of held lengths in sorted order
  int64_t* gpos[2];          // [N] FLAT: offset of sequence i in its group's token stream
  int32_t* pos[2];           // [N] THRESHOLD: position of sequence i in its group
  int64_t* pbase;            // [N+1] piece base per sequence
  // pieces (unsorted, then sorted by key)
  int32_t* pc_i; int32_t* pc_x; int32_t* pc_y; int32_t* pc_kk;  // kk = ks | kd<<8 | key<<16
  int32_t* ps_i; int32_t* ps_x; int32_t* ps_y; int32_t* ps_kk;
  int64_t* ps_scan;          // [max_pieces+1]
  int64_t* cta_sums;         // [kMaxPlanGrid] grid-scan partials
  int32_t* ghist;            // [kMaxPlanGrid][kMaxKeys] grid-partition histograms
  int64_t* vtmp;             // [max(N, max_pieces) + 1] scan inputs
  int32_t* ktmp;             // [max(N, max_pieces)] partition keys
  int32_t* ptmp;             // [max(N, max_pieces)] partition output (position -> index)
  int64_t* fhist;            // SP = 1 fast path: [2][kMaxPlanGrid][kMaxKeys + 2 kMaxShards]
  uint64_t* phase_ts;        // debug (EARL_PLAN_TRACE): %globaltimer at phase boundaries
  int64_t max_pieces;
  int64_t max_records;
  Records rec;
};

struct PeerPads {
  uint64_t* p[kMaxWorld];
};
struct McTeams {             // NEXT-3: per dst shard, the multicast address of its team (0: none)
  uint64_t va[kMaxShards];
  uint32_t mask[kMaxShards];  // the team's ranks
};
struct RecvOffsets {
  uint64_t v[kMaxFields];   // window-relative receive offsets of this rank (kNoOffset = NULL)
};

enum CopyMode { kDirect = 0, kPack = 1, kUnpack = 2 };

struct CopyArgs {
  int32_t mode;
  int32_t n_fields;
  int32_t view_rank;       // -1: every record (emulated); else records of source rank view_rank
  int32_t nts;             // min(tp_src, tp_dst)
  int32_t rank0_s, tp_s, rank0_d, tp_d, sp_d, n_dst_shards, n_src_shards;
  int32_t protocol;        // 1: multi-process fused exec (epoch release / acquire at the end)
  int32_t remote_tma;      // 1: peer replicas by bulk TMA stores too (EARL_REMOTE_STORE=tma)
  int32_t mc_on;           // NEXT-3: some dst shard's replicas form a multicast team with this rank
  uint32_t peer_mask;      // ranks taking part in the completion protocol (a node's, NEXT-4)
  uint32_t ds_mask;        // pack (real rank): destination shards to pack (~0: all)
  uint32_t src_mask;       // unpack (real rank): source ranks whose messages are in recv_stage
  uint8_t* const* mc_tab;  // [kMaxShards][kMaxFields] multicast bases (entry barrier), protocol 1
  const uint8_t* recv_stage;                  // unpack on a real rank: received messages
  uint32_t Bf[kMaxFields];
  uint64_t Bpre[kMaxFields + 1];  // prefix of Bf
  const PlanHeader* hdr;
  Records rec;
  const uint8_t* src[kMaxWorld][kMaxFields];  // per source comm rank (direct/pack)
  uint8_t* dst[kMaxWorld][kMaxFields];        // per destination comm rank (direct/unpack)
  uint8_t* stage[kMaxWorld];                  // per source comm rank (pack dst / unpack src)
  // completion protocol for a multi-process comm (view_rank >= 0 && world > 1)
  int32_t world;
  int32_t me;
  unsigned int* done_ctr;                     // device counter for the last-CTA pattern
  uint64_t* my_pad;                           // this rank's signal pad (local)
  uint64_t* peer_pad[kMaxWorld];              // peers' signal pads (mapped)
  uint8_t* const* dst_tab;                    // protocol 1: [kMaxWorld][kMaxFields] destination
                                              // field bases resolved by the entry barrier from
                                              // every destination's published window offsets
  uint64_t timeout_ns;
  int32_t* err;                               // where to latch TIMEOUT (plan header)
  int32_t* err_detail;
  uint64_t* trace;                            // debug: per-warp (t_start, t_end, bytes, chunks)
  unsigned int* work_ctr;                     // plan-owned dynamic scheduling counters
  unsigned int* fin_ctr;
};

// signal pad slots (uint64 each): [0, 8) ready flags written by peer p at p; [8, 16) done flags
// (2 * epoch + failed: a peer that skipped its copies says so); [16] this rank's exec epoch;
// [32, 48) this rank's published receive offsets (one per field, window-relative, kNoOffset =
// NULL), read by every peer after it acquires this rank's ready flag; [64, 192) the destination
// table [kMaxWorld][kMaxFields] this rank's entry barrier resolved from the peers' offsets.
constexpr int kReadySlot = 0;
constexpr int kDoneSlot = 8;
constexpr int kEpochSlot = 16;  // this rank's exec epoch (written by its own entry barrier)
constexpr int kLensEpochSlot = 17;  // this rank's length-gather epoch (a1)
constexpr int kLensSlot = 24;       // [24, 32): length-gather flags written by peer p at p
constexpr int kOffSlot = 32;
constexpr int kDstTabSlot = 64;
constexpr int kMcTabSlot = 192;  // [192, 320): multicast bases [kMaxShards][kMaxFields] (NEXT-3)
constexpr uint64_t kNoOffset = ~0ull;

// step a1 (lengths.cu): the device gather of the global length vector
struct LensArgs {
  int32_t world, me, emulated;
  int64_t cap;                      // sequences per gather buffer (multi-process)
  int64_t total;                    // sum of counts
  int64_t counts[kMaxWorld];
  int64_t start[kMaxWorld];         // exclusive prefix of counts
  const int32_t* local;             // this rank's lengths (multi-process)
  const int32_t* src[kMaxWorld];    // every rank's lengths (emulated)
  int32_t* out;                     // [total]
  uint64_t* my_pad;
  uint64_t* peer_pad[kMaxWorld];    // window bases (pad first, then the gather areas)
  unsigned int* ctr;                // last-CTA counter (comm-owned)
  int32_t* err;                     // comm-owned [2]: status, detail (missing-peer mask)
  uint64_t timeout_ns;
};

__device__ __forceinline__ void st_release_sys_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// NEXT-2 (aggregate.cu): returns / advantages on the source ranks (SP = 1)
// returns_kernel look-back state: one descriptor per token window of a source rank.  Each word
// is {tag << 32 | float bits}, tag = (epoch << 2) | kind, written with one 64-bit store and
// validated on its own by the reader: no fences between the value and its flag.
struct AggWindow {
  uint64_t S;    // kind 1: the window's map x -> S + P x ...
  uint64_t P;    // ... (both words must carry the current tag)
  uint64_t inc;  // kind 2: G at the window's first token
  uint64_t pad;
};
struct AggWork {
  uint32_t work_ctr;  // window / unit claims (reset by the last CTA)
  uint32_t fin_ctr;   // finished CTAs
  uint32_t epoch;     // launches so far: flags of older launches never match
  uint32_t pad;
};
#ifndef EARL_UNIT_TOK
#define EARL_UNIT_TOK 8192
#endif
constexpr int kUnitTok = EARL_UNIT_TOK;  // returns unit kernel: a unit = the sequences starting in [k*kUnitTok, (k+1)*kUnitTok)
constexpr int64_t kUnitMaxLen = int64_t(1) << 17;  // ... used when no sequence is longer than this
// The unit kernel pays off when the batch has no very long sequence (one warp streams a unit)
// and enough units to keep every warp busy: at least kUnitsPerWarp units per resident warp
// (measured with 4096-token units: C5-lt, 83K units, 0.60 ms against 0.71 windowed; C2, 322
// units, 54 against 24 us).
constexpr int64_t kUnitsPerWarp = 4;
constexpr int kUnitWarpsPerSm = 16;  // returns_units_kernel: 2 CTAs x 8 warps
// The unit kernel keeps positions inside a rank buffer in int32: ranks of at most kU2MaxTok tokens.
constexpr int64_t kU2MaxTok = (int64_t(1) << 31) - 4 * kUnitTok;
__host__ __device__ inline bool prefer_units(int64_t max_len, int64_t units, int64_t warps,
                                             int64_t max_rank_tokens) {
  return max_len <= kUnitMaxLen && units >= kUnitsPerWarp * warps && max_rank_tokens <= kU2MaxTok;
}
// The cooperative returns kernel: one window of 512 * nb tokens (nb = 1, 2 or 4) per warp of a
// co-resident grid, so a batch fits when its windows do not outnumber the grid's warps.
constexpr int kCoopMaxNB = 4;
// Returns kernels (AggArgs::gate = id + 1 runs a kernel only if the device's choice is id).
enum ReturnsKernel { kRetUnits = 0, kRetWindows = 1, kRetCoop = 2 };
// Which returns kernel a batch gets, from its source ranks' token counts (host and device
// evaluate the same rule): the cooperative kernel when every window gets its own warp, the
// unit kernel for large batches without very long sequences, else the windowed look-back kernel.
// *coop_nb: the cooperative kernel's batches per window (0: does not fit).
__host__ __device__ inline int choose_returns(const int64_t* ntok, int n, int64_t max_len,
                                              int64_t unit_warps, int64_t coop_warps,
                                              int* coop_nb) {
  int64_t units = 0, big = 0, cw[3] = {0, 0, 0};
  for (int i = 0; i < n; ++i) {
    units += (ntok[i] + kUnitTok - 1) / kUnitTok;
    big = ntok[i] > big ? ntok[i] : big;
    for (int k = 0; k < 3; ++k) cw[k] += (ntok[i] + (512 << k) - 1) / (512 << k);
  }
  int nb = 0;
  for (int k = 0; k < 3 && nb == 0; ++k)
    if (cw[k] <= coop_warps) nb = 1 << k;
  if (coop_nb) *coop_nb = nb;
  if (nb > 0) return kRetCoop;
  return prefer_units(max_len, units, unit_warps, big) ? kRetUnits : kRetWindows;
}

struct AggArgs {
  AggWork* ws;
  AggWindow* win;
  int64_t win_cap;
  int64_t* unit_first;     // unit kernel: first sequence (sorted position) of every unit
  int32_t gate;            // 0: run; 1: run only if the unit kernel is preferred; 2: only if not
  int64_t resident_warps;  // the unit kernel's resident warps (prefer_units)
  int64_t coop_warps;      // the cooperative kernel's warps (its grid; 0: not available)
  int32_t coop_nb;         // its batches per window (0: the kernel decides from the plan header)
  PlanArgs plan;
  const PlanHeader* hdr;
  int32_t world;
  int32_t view_rank;       // -1: every source rank (emulated comm); else this rank
  float gamma, eps;
  float gamma16;            // gamma^16 (product of 16 fp32 factors, as a lane of 16 tokens)
  float gpw[5];             // gamma^(16 * 2^k), k = 0..4 (gpw[0] = gamma16, then squares)
  float g4, g512;           // gamma^4 (a 4-token chunk), gamma^512 (a 512-token batch)
  const float* rewards[kMaxWorld];   // per source comm rank: token rewards (fp32)
  const uint8_t* mask[kMaxWorld];    // token mask (u8, 1 = counted)
  float* returns[kMaxWorld];         // token returns G (fp32)
  float* adv[kMaxWorld];             // token advantages A (fp32)
  float* seq_return[kMaxWorld];      // per-sequence return G_0 (fp32), optional
  double* partial;                   // [3] sum m, sum m G, sum m G^2 (accumulated)
  const double* stats;               // [3] the same over the whole batch (after the all-reduce)
};

// Delay injection (SURVEY.md §5 race detection; build with EARL_NVCC_DEFINES=EARL_DELAY_INJECT=1):
// a pseudo-random spin of up to ~20 us per (CTA, warp, site) at the points where flag ordering
// or look-back correctness depends on timing, so tests shake out missing fences and waits.
#ifndef EARL_DELAY_INJECT
#define EARL_DELAY_INJECT 0
#endif
__device__ __forceinline__ void delay_inject(uint32_t site) {
  if (EARL_DELAY_INJECT) {
    uint32_t x = blockIdx.x * 2654435761u ^ (threadIdx.x >> 5) * 40503u ^ site * 2246822519u;
    x ^= x >> 15; x *= 0x2c1b3c6du; x ^= x >> 12; x *= 0x297a2d39u; x ^= x >> 15;
    const long long cycles = (long long)(x % 40000u);  // up to ~20 us at 1.9 GHz
    const long long t0 = clock64();
    while (clock64() - t0 < cycles) {}
  }
}

// Opt a kernel in to `bytes` of dynamic shared memory on the current device.  The attribute is
// per device, so a process driving several GPUs opts in once on each (done[] per device id).
template <class F>
inline cudaError_t opt_in_dynamic_smem(F* func, int bytes, bool (&done)[64]) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const bool tracked = dev >= 0 && dev < 64;
  if (tracked && done[dev]) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess && tracked) done[dev] = true;
  return e;
}

// NEXT-3 (vmm.cu): cuMemCreate windows shared by POSIX file descriptor, NVLS multicast teams
struct VmmMem {
  uint64_t handle;  // CUmemGenericAllocationHandle
  uint64_t va;      // mapped address in this process (0: not mapped)
  uint64_t size;
  int32_t fd;       // exported descriptor (-1: none)
};
bool vmm_available();
bool multicast_entry_points();
bool vmm_create(int device, uint64_t bytes, VmmMem* out, const char** why);
bool vmm_export(VmmMem* m, int32_t* fd, const char** why);
bool vmm_import(int device, int32_t pid, int32_t fd, uint64_t size, VmmMem* out, const char** why);
void vmm_free(VmmMem* m);
bool mc_create(int n_devices, uint64_t size, VmmMem* out, const char** why);
bool mc_import(int32_t pid, int32_t fd, uint64_t size, VmmMem* out, const char** why);
bool mc_join(VmmMem* mc, int device, const VmmMem& window, const char** why);
void mc_free(VmmMem* mc, int device);

// launchers (defined in the .cu files)
cudaError_t launch_returns(const AggArgs& a, int sm_count, cudaStream_t s);
cudaError_t launch_returns_units(const AggArgs& a, int sm_count, cudaStream_t s);
int returns_coop_capacity_warps(int sm_count);  // co-resident warps of the cooperative kernel
cudaError_t launch_returns_coop(const AggArgs& a, int64_t windows, int sm_count, cudaStream_t s);
int64_t returns_windows(int64_t tokens);
cudaError_t launch_advantages(const AggArgs& a, int sm_count, int64_t tokens, cudaStream_t s);
int planner_grid(int64_t n_seqs, int64_t max_pieces, int sm_count, size_t lpt_smem, bool fast);
cudaError_t launch_planner(const PlanArgs& a, size_t lpt_smem, int grid, bool fast, cudaStream_t s);
cudaError_t launch_copy(const CopyArgs& a, int sm_count, int shape, cudaStream_t s);
cudaError_t launch_entry_barrier(uint64_t* my_pad, uint64_t* const* peer_pad, int world,
                                 uint32_t peers, int me, int n_fields, const uint64_t* recv_off,
                                 const McTeams& mct, uint64_t timeout_ns, int32_t* err,
                                 int32_t* err_detail, cudaStream_t s);
cudaError_t launch_gather_lengths(const LensArgs& a, int sm_count, cudaStream_t s);
cudaError_t launch_fill_i32(int32_t* p, int32_t v, int64_t n, cudaStream_t s);
cudaError_t launch_local_meta(const PlanArgs& a, int rank_g, int rank_k, int32_t* cu, int64_t* ids,
                              int32_t* tok_start, cudaStream_t s);

}  // namespace earl
