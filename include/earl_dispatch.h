/*
 * earl_dispatch.h -- C ABI of the B200-native EARL data dispatcher.
 *
 * What it does (§2 "Data Dispatcher"): intermediate RL batches --
 * variable-length sequences carrying per-token fields ("tokens, log-probabilities, rewards,
 * returns, and other tensors") -- held by the ranks of one parallel layout
 * are re-distributed to the ranks of another layout, "adaptive to the current data
 * distribution layout and parallelism configuration", by sending "data
 * directly to the target workers from their computation origins": an
 * all-to-all instead of the centralized all-gather-and-scatter.
 *
 * The two calls named by the build's north star are earl_dispatch_plan (device-side
 * planner: prefix sums over lengths, length-balanced assignment, SP chunking, per-segment
 * offsets) and earl_dispatch_exec (one fused pass: read each source byte once, store it at
 * its final offset on every destination replica, over NVLink peer mappings).
 * earl_dispatch_pack / earl_dispatch_unpack are the staged alternative (gather into
 * contiguous per-destination-shard messages, scatter from them).  Readings of the paper
 * are listed in DESIGN.md; the ones that shape this ABI are
 * repeated at the declarations.
 *
 * Conventions
 *  - Every call returns an earl_status_t; outputs go through out-parameters.  On error,
 *    earl_last_error() (thread-local) holds a one-line message.
 *  - Device work is stream-ordered and asynchronous.  `stream` is a cudaStream_t passed
 *    as void* (NULL = legacy default stream).  Errors found on the device (negative
 *    length, EXPLICIT group out of range, int32 overflow of cu_seqlens, peer timeout) are
 *    latched in the plan and reported by the next host-synchronising call
 *    (earl_plan_local_sizes, earl_plan_stats, earl_plan_export, earl_plan_sync).
 *  - Collective semantics (like NCCL): in a multi-process comm every rank calls
 *    earl_dispatch_plan / earl_dispatch_exec in the same order with identical layouts,
 *    lengths and fields.  Each rank computes the same plan independently (integer-only,
 *    deterministic); no metadata is exchanged.  A rank in neither layout participates
 *    with zero bytes.
 *  - Emulated comm (rank == EARL_ALL_RANKS): one process holds all `world` ranks on one
 *    device; buffer arrays are then rank-major [world][n_fields] and one launch serves
 *    all ranks (the 1-GPU measurement mode of SURVEY.md §8(d)).
 *  - Field base pointers must be 16-byte aligned (cudaMalloc gives 256 B), else
 *    EARL_ERR_INVALID_ARGUMENT.  Field bytes are opaque and never interpreted (reading
 *    c10): the result is bit-exact.
 *  - A comm is not thread-safe.  Planning is pure: the same inputs give the same plan.
 *
 * Ownership: the caller owns send/recv/stage buffers, seq_lens and streams.  The plan owns
 * its device metadata (freed by earl_plan_destroy after the plan's stream work).  The comm
 * owns its symmetric window, the peer mappings and the signal pad.
 */
#ifndef EARL_DISPATCH_H_
#define EARL_DISPATCH_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define EARL_API __attribute__((visibility("default")))
#else
#define EARL_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define EARL_ABI_VERSION 3
#define EARL_MAX_WORLD 8        /* reading c21: one box, W <= 8 */
#define EARL_MAX_FIELDS 16
#define EARL_HANDLE_BYTES 128   /* size of the exported window handle */
#define EARL_ALL_RANKS (-1)     /* emulated comm: this process holds every rank */
#define EARL_LPT_MAX_SEQS 8192  /* reading c4: LPT sorts in one CTA's shared memory */

typedef enum {
  EARL_OK = 0,
  EARL_ERR_INVALID_ARGUMENT = 1, /* null/misaligned pointer, L_i < 0, bad enum, n_fields > 16 */
  EARL_ERR_LAYOUT = 2,           /* dp*sp*tp ranks outside the comm, sum(counts) != N,
                                    EXPLICIT group outside [0, dp)        */
  EARL_ERR_CAPACITY = 3,         /* window too small, dst rank > INT32_MAX tokens (c12),
                                    LPT with N > 8192, buffer too small                  */
  EARL_ERR_CUDA = 4,             /* a CUDA runtime call failed                            */
  EARL_ERR_NCCL = 5,             /* an NCCL call of the staged exchange failed (K8)       */
  EARL_ERR_TIMEOUT = 6,          /* peer signals missing; mask in earl_last_error */
  EARL_ERR_MISMATCH = 7,         /* plan hash differs across ranks (debug)                */
  EARL_ERR_UNSUPPORTED = 8,      /* world > 8, wrong comm kind for the call               */
  EARL_ERR_POLICY = 9            /* selector: a context range with no OOM-free configuration,
                                    or an average length outside every range                */
} earl_status_t;

typedef enum {
  EARL_ASSIGN_GIVEN_COUNTS = 0, /* group g holds seqs [sum_{h<g} counts[h], +counts[g])        */
  EARL_ASSIGN_CONTIG = 1,       /* g(i) = min(D-1, floor(D*(2*P_i+L_i)/(2*T))), T==0 -> blocks */
  EARL_ASSIGN_LPT = 2,          /* Graham LPT: (L desc, i asc) to least-loaded group, ties low */
  EARL_ASSIGN_EXPLICIT = 3      /* g(i) = group_of_seq[i]                                    */
} earl_assign_t;

/* How an SP group splits its sequences' tokens (readings c7, n1-n3). */
typedef enum {
  EARL_SP_BLOCK = 0,     /* SP rank k holds BLOCK chunk k = [k*q+min(k,r), (k+1)*q+min(k+1,r)),
                            q = L/sp, r = L%sp, of every sequence (reading c7)               */
  EARL_SP_ZIGZAG = 1,    /* 2*sp BLOCK chunks; rank k holds chunks k and 2*sp-1-k (ring-attention
                            / context-parallel load balance, reading n1)                      */
  EARL_SP_FLAT = 2,      /* the group's sequences concatenated (ascending i) into one stream,
                            BLOCK-split over the sp ranks, no padding (Ulysses, reading n2)   */
  EARL_SP_THRESHOLD = 3  /* sequences with L >= sp_min_len are BLOCK-split; shorter ones go whole
                            to SP rank (position in group) mod sp (reading n3)                */
} earl_sp_split_t;

/* A parallel layout (reading c1/c3): ranks rank0 .. rank0+dp*sp*tp-1 of the comm, with
 * rank(g,k,t) = rank0 + (g*sp + k)*tp + t  (TP fastest, then SP, then DP).
 * DP group g holds the sequences assigned to it in ascending global index (reading c5);
 * its SP rank k holds, of every such sequence, the tokens the sp_split rule gives it, in
 * ascending position; every TP rank of (g,k) holds a full copy (reading c2).  When the source
 * has several TP replicas, dst replica td is fed by source replica td mod tp_src (reading c9). */
typedef struct {
  int32_t rank0, dp, sp, tp;
  int32_t assign;               /* earl_assign_t */
  int32_t sp_split;             /* earl_sp_split_t */
  int32_t sp_min_len;           /* EARL_SP_THRESHOLD: shortest sequence that is split (>= 0) */
  int32_t reserved;             /* 0 */
  const int64_t* counts;        /* HOST [dp], GIVEN_COUNTS only */
  const int32_t* group_of_seq;  /* DEVICE [N], EXPLICIT only; read by the planner at every
                                   earl_dispatch_plan / earl_plan_replan, so it must stay valid
                                   for the plan's lifetime */
} earl_layout_t;

/* One per-token field: bytes_per_elem * elems_per_token bytes per token (opaque). */
typedef struct {
  uint32_t bytes_per_elem, elems_per_token;
} earl_field_t;

typedef struct earl_comm* earl_comm_t;
typedef struct earl_plan* earl_plan_t;

typedef struct {
  int32_t world;
  int32_t n_fields;
  uint64_t bytes_per_token;               /* B = sum_f B_f */
  uint64_t total_tokens;                  /* T */
  uint64_t C[EARL_MAX_WORLD][EARL_MAX_WORLD]; /* payload bytes rank s -> rank d (per replica) */
  uint64_t egress[EARL_MAX_WORLD];        /* sum_{d != s} C[s][d]   (NVLink out)            */
  uint64_t ingress[EARL_MAX_WORLD];       /* sum_{s != d} C[s][d]   (NVLink in)             */
  uint64_t self_bytes[EARL_MAX_WORLD];    /* C[r][r]: local copy                            */
  uint64_t total_bytes, moved_bytes, max_egress, max_ingress;
  uint64_t read_bytes[EARL_MAX_WORLD];    /* fused exec: source bytes read once per rank     */
  uint64_t stage_bytes[EARL_MAX_WORLD];   /* packed message buffer size per source rank      */
  int64_t n_local_seqs[EARL_MAX_WORLD];   /* per destination rank (0 if not in dst layout)   */
  int64_t n_local_tokens[EARL_MAX_WORLD];
  int64_t n_segments;                     /* canonical (uncoalesced) records incl. replicas  */
  int64_t n_pieces;                       /* (sequence, overlap) pieces before replication   */
  int64_t n_records;                      /* copy records (piece x sending replica)          */
} earl_plan_stats_t;

/* ---- comm -------------------------------------------------------------------------- */

/* Create a comm.  rank in [0, world) for one process per GPU, or EARL_ALL_RANKS to emulate
 * all ranks in this process on `cuda_device`.  window_bytes: size of this rank's symmetric
 * receive window (per emulated rank in emulated mode); P2P exec writes into it.
 * Errors: UNSUPPORTED (world outside [1,8]), INVALID_ARGUMENT, CUDA. */
EARL_API earl_status_t earl_comm_create(int32_t rank, int32_t world, int32_t cuda_device,
                               uint64_t window_bytes, earl_comm_t* comm);
/* Multi-process bootstrap: export this rank's window handle (EARL_HANDLE_BYTES bytes),
 * all-gather them out of band (e.g. torch.distributed), then import all `world` handles
 * (rank-major).  Importing maps every peer's window (CUDA IPC over NVLink P2P). */
EARL_API earl_status_t earl_comm_export_handle(earl_comm_t comm, void* handle_out);
EARL_API earl_status_t earl_comm_import_peers(earl_comm_t comm, const void* handles);
/* Collective bump allocation inside the window: every rank calls it with the same sizes in
 * the same order and gets the same offset, so peers address it as base_peer + offset.
 * In emulated mode `rank` selects the emulated rank's window; otherwise it is ignored.
 * Errors: CAPACITY when the window is exhausted. */
EARL_API earl_status_t earl_comm_alloc(earl_comm_t comm, int32_t rank, uint64_t bytes, void** dev_ptr);
EARL_API earl_status_t earl_comm_reset_alloc(earl_comm_t comm);
EARL_API earl_status_t earl_comm_info(earl_comm_t comm, int32_t* rank, int32_t* world, int32_t* emulated);
EARL_API earl_status_t earl_comm_destroy(earl_comm_t comm);
/* Bit p of *mask is set when peer p's window is mapped into this process (CUDA IPC; bench
 * evidence of the N-rank data plane).  Emulated comm: 0. */
EARL_API earl_status_t earl_comm_peer_mask(earl_comm_t comm, uint32_t* mask);

/* NEXT-3: NVLS multicast for TP-replicated destinations.  With EARL_NVLS=1 in
 * the environment at earl_comm_create, a multi-process comm allocates its window with cuMemCreate
 * (exported as a POSIX file descriptor that peers fetch with pidfd_getfd; export/import as
 * above) and can bind it to multicast teams.  A team is a set of ranks (bit mask), normally the
 * TP replicas of one destination shard: the lowest rank of the team calls earl_comm_mc_create
 * (cuMulticastCreate over popcount(mask) devices; *handle_out, EARL_HANDLE_BYTES, to broadcast),
 * then every rank of the comm calls earl_comm_mc_join with that handle (members add their device,
 * bind their whole window at multicast offset 0 and map the multicast address -- concurrently:
 * the bind waits for every member; other ranks return at once).  An exec whose destination shard
 * has a team containing the sending rank, whose source layout has tp == 1 and whose members put
 * the field at the same window offset stores the 16-B interior of each record once with
 * multimem.st (NVSwitch writes every replica) instead of once per replica; heads and tails and
 * everything else stay unicast.  Errors: UNSUPPORTED (no EARL_NVLS window, or the driver / device
 * cannot create the team -- e.g. a box with one visible GPU), INVALID_ARGUMENT, CAPACITY (> 8
 * teams). */
/* NEXT-4 ("further gains with RDMA"): a comm spanning several
 * nodes of node_size consecutive ranks each (node n = ranks [n*node_size, (n+1)*node_size)).  Call
 * before earl_comm_import_peers: only same-node windows are mapped.  Then, on this comm:
 *   earl_dispatch_exec        moves the records whose destination replica is on this node (fused
 *                             P2P; the barrier and done flags involve the node's ranks only);
 *   earl_dispatch_pack / earl_plan_messages / earl_dispatch_exchange / earl_dispatch_unpack /
 *   earl_dispatch_exec_staged cover exactly the messages between nodes (pack: the destination
 *                             shards with a replica on another node; unpack: the messages from
 *                             other nodes' ranks, concatenated in source-rank order);
 *   earl_dispatch_exec_hier   does both: fused P2P inside the node, then the NCCL exchange
 *                             (earl_comm_init_nccl: NCCL picks IB / RoCE between nodes).
 * The two legs write disjoint parts of the receive arrays.  earl_allgather_lengths is
 * UNSUPPORTED on such a comm (gather the lengths over the process group).
 * Errors: INVALID_ARGUMENT (node_size does not divide the world, or peers already imported),
 * UNSUPPORTED (emulated comm). */
EARL_API earl_status_t earl_comm_set_nodes(earl_comm_t comm, int32_t node_size);
/* The NVLink options of the multi-process fused exec, for choosing by measurement (the bench's
 * N > 1 tuning pass): remote_store 0 = peer replicas by 16-B warp stores, 1 = by bulk TMA stores
 * to the peer address, -1 = EARL_REMOTE_STORE's choice (warp stores by default); p2p_shape = a
 * copy-engine shape id (1-8, 11, 14; e.g. 3 = 8 warps x 3 stages x 8 KB, 14 = 2 x 2 x 16 KB), or
 * -1 = EARL_COPY_CFG_P2P's choice (else chosen from the field widths).  Bytes moved are identical
 * for every setting.  Errors: INVALID_ARGUMENT. */
EARL_API earl_status_t earl_comm_set_exec_options(earl_comm_t comm, int32_t remote_store,
                                                  int32_t p2p_shape);
EARL_API earl_status_t earl_dispatch_exec_hier(earl_plan_t plan, const void* const* send_bufs,
                                               void* const* recv_bufs, void* stream);

EARL_API earl_status_t earl_comm_mc_create(earl_comm_t comm, uint32_t team_mask, void* handle_out);
EARL_API earl_status_t earl_comm_mc_join(earl_comm_t comm, uint32_t team_mask, const void* handle);

/* Step a1: the global length vector every rank plans from (the layout
 * knowledge of PAPER.md:178), gathered on the device.  Global order is rank-major (reading c6):
 * rank r's counts[r] lengths occupy [sum_{q<r} counts[q], +counts[r]) of the output.
 * counts: HOST [world], identical on every rank (the source layout's per-rank sequence counts,
 *   e.g. rollout GIVEN_COUNTS; 0 for replicas that hold no sequences of their own).
 * local_lens: [1] (emulated: [world]) DEVICE int32 pointers to this rank's counts[rank] lengths
 *   (NULL where the count is 0).
 * global_lens: DEVICE int32 [sum(counts)] output, written on `stream`.
 * Collective in a multi-process comm: one kernel stores this rank's lengths into every peer's
 * gather area (a double buffer after the window's signal pad, EARL_LENS_CAPACITY sequences,
 * default 2^18, read at earl_comm_create), releases an epoch flag to each peer and acquires
 * theirs; no host synchronisation, so gather + earl_plan_replan + earl_dispatch_exec capture
 * into one CUDA graph.  A peer missing for longer than the comm's timeout latches TIMEOUT,
 * reported by earl_comm_check.
 * Errors: INVALID_ARGUMENT (NULL, negative count), CAPACITY (sum(counts) > the gather area). */
EARL_API earl_status_t earl_allgather_lengths(earl_comm_t comm, const int64_t* counts,
                                              const void* const* local_lens, int32_t* global_lens,
                                              void* stream);
/* Synchronise `stream` and report (then clear) an error latched on the device by a comm-level
 * collective (earl_allgather_lengths: TIMEOUT with the missing peers' bit mask). */
EARL_API earl_status_t earl_comm_check(earl_comm_t comm, void* stream);

/* ---- plan -------------------------------------------------------------------------- */

/* Plan the dispatch of N sequences from layout `src` to layout `dst`.
 * seq_lens: DEVICE int32 [N], global index order (reading c6); L_i = 0 allowed (c11),
 * L_i < 0 latches INVALID_ARGUMENT (c20).  fields: HOST [n_fields] (<= 16).
 * Computes on `stream`, without a host synchronisation: P = exclusive scan of L (int64);
 * g_src(i), g_dst(i); per-rank local token offsets; every (sequence, overlap, replica)
 * segment with its source, destination and message offsets; per-(rank, shard) message
 * sizes; destination metadata.  Host-side checks: layout validity (LAYOUT), N <= 8192 for
 * LPT (CAPACITY), n_fields (INVALID_ARGUMENT).  The plan owns its device memory. */
EARL_API earl_status_t earl_dispatch_plan(earl_comm_t comm, const earl_layout_t* src,
                                 const earl_layout_t* dst, const int32_t* seq_lens,
                                 int64_t n_seqs, const earl_field_t* fields, int32_t n_fields,
                                 void* stream, earl_plan_t* plan);
/* Re-plan the same N sequences (same comm, layouts, fields) for new lengths seq_lens (DEVICE
 * int32 [N]; ignored, may be NULL, for a plan from earl_plan_seq_fields, which re-reads its
 * token plan's groups) into the plan's existing device memory: nothing is allocated, so a training loop
 * re-plans every batch at the planner's cost only.  Stream-ordered: work still using the
 * previous plan must precede it on `stream` (or be synchronised).  earl_dispatch_plan followed
 * by earl_plan_replan / earl_dispatch_exec is capturable into a CUDA graph; after replaying one,
 * synchronise the stream before host queries (earl_plan_stats, ...). */
EARL_API earl_status_t earl_plan_replan(earl_plan_t plan, const int32_t* seq_lens, void* stream);
/* Wait for the plan and report device-latched errors. */
EARL_API earl_status_t earl_plan_sync(earl_plan_t plan);
/* Destination rank `rank`'s holding (host; synchronises): sequences and tokens. */
EARL_API earl_status_t earl_plan_local_sizes(earl_plan_t plan, int32_t rank, int64_t* n_local_seqs,
                                    int64_t* n_local_tokens);
/* Destination metadata of rank `rank` written to DEVICE buffers on `stream`:
 * cu_seqlens int32 [n_local_seqs+1], seq_ids int64 [n_local_seqs] (global index),
 * tok_start int32 [n_local_seqs] (first token this rank holds of the sequence, i.e. the start
 * of its first chunk; for ZIGZAG the second chunk starts at L - (its length)).
 * Any pointer may be NULL to skip it. */
EARL_API earl_status_t earl_plan_local_meta(earl_plan_t plan, int32_t rank, int32_t* cu_seqlens,
                                   int64_t* seq_ids, int32_t* tok_start, void* stream);
/* The plan's group assignment g(i) of every sequence under src and dst (DEVICE int32 [N]
 * outputs, either may be NULL), stream-ordered.  Used to route per-sequence fields (rewards,
 * returns) with their sequences: a second plan over unit lengths with these groups as EXPLICIT
 * layouts and the SP degree folded into TP (reading n4). */
EARL_API earl_status_t earl_plan_groups(earl_plan_t plan, int32_t* src_groups, int32_t* dst_groups,
                                        void* stream);
/* Reading n4: plan the routing of PER-SEQUENCE fields (a reward or score per
 * episode, n_fields of them, bytes_per_elem * elems_per_token bytes per SEQUENCE) along
 * `token_plan`: every destination rank (g, k, t) receives one record per sequence of its group,
 * in the group order of the token plan (every SP rank and TP replica holds a copy), sent by the
 * source rank (g_src(i), SP 0, t mod tp_src).  Built on the device as a second plan over unit
 * lengths whose layouts are the token plan's with SP folded into TP and the groups pinned as
 * EXPLICIT (its own copies of g_src / g_dst, refreshed by earl_plan_replan(seq_plan, NULL, s)
 * after the token plan is re-planned).  Execute with earl_dispatch_exec (buffers hold one record
 * per sequence); query with the usual calls.  The token plan stays alive until the last plan
 * made from it is destroyed.  Errors: as earl_dispatch_plan; INVALID_ARGUMENT if token_plan is
 * itself a per-sequence plan. */
EARL_API earl_status_t earl_plan_seq_fields(earl_plan_t token_plan, const earl_field_t* fields,
                                            int32_t n_fields, void* stream, earl_plan_t* seq_plan);
/* Byte accounting of SPEC.md:239-247 (host; synchronises). */
EARL_API earl_status_t earl_plan_stats(earl_plan_t plan, earl_plan_stats_t* stats);
/* Debug check of replicated planning (every rank computes a byte-identical plan
 * with no metadata exchange): a 64-bit FNV-1a hash of the plan's tables and its record arrays
 * (host; synchronises; copies the records to the host, so O(records) time).  Equal inputs give
 * equal hashes on every rank; the binding all-gathers them and reports EARL_ERR_MISMATCH. */
EARL_API earl_status_t earl_plan_hash(earl_plan_t plan, uint64_t* hash);
/* Debug: the canonical, uncoalesced segment table in (s, d, i, x) order (reading c19),
 * one record per (sequence i, token overlap [x,y), destination replica): source rank s,
 * destination rank d, source local token offset, destination local token offset.
 * Pass capacity 0 / NULL arrays to query n_segments only (host; synchronises). */
EARL_API earl_status_t earl_plan_export(earl_plan_t plan, int64_t capacity, int64_t* n_segments,
                               int32_t* s, int32_t* d, int64_t* seq, int32_t* x, int32_t* y,
                               int64_t* src_off, int64_t* dst_off);
EARL_API earl_status_t earl_plan_destroy(earl_plan_t plan);

/* ---- execution --------------------------------------------------------------------- */

/* Fused dispatch (SURVEY.md §8(a) a6 + a7): every source byte is read once and stored at
 * its final offset on every destination replica.
 * send_bufs: field arrays this rank holds under `src` ([n_fields]; emulated:
 *   [world][n_fields], rank-major), each n_src_tokens(rank) * B_f bytes, 16-B aligned.
 *   DEVICE memory, or page-locked HOST memory mapped into the device address space
 *   (cudaHostAlloc / cudaHostRegister under UVA): the kernel then reads it over PCIe itself
 *   (zero-copy; no separate host-to-device copy).
 * recv_bufs: DEVICE field arrays under `dst`, sized n_local_tokens * B_f; NULL = this rank
 *   receives nothing for that field (e.g. it is in no destination layout).  Multi-process comm
 *   with world > 1: each non-NULL one must lie inside this rank's window (earl_comm_alloc) --
 *   peers store into it over NVLink.  Offsets need not match across ranks: every rank
 *   publishes its own offsets in its signal pad and the senders write where the destination
 *   put its buffers, so a source-only rank passing NULLs still sends all of its records.
 * Protocol (multi-process): entry barrier (every peer's stream reached exec, so its recv
 * buffers may be overwritten; each rank's receive offsets are published with its ready flag),
 * stores, system-scope fence, release of a done flag (2 * epoch + failed) into each peer's
 * signal pad, acquire-wait for every peer's.  When the stream passes the call, this rank's
 * recv buffers are complete.  A peer missing for > 10 s (or the EARL_TIMEOUT_MS read at
 * earl_comm_create) latches TIMEOUT with the bit mask of the missing peers; a peer that skipped
 * its copies (its own barrier timed out) makes every rank that sees it latch TIMEOUT naming it
 * (detail bits 8-15).  Both are reported by the next synchronising call (a
 * barrier timeout names the missing workers).
 * Launches on one plan are serialised in issue order across streams (each waits for the plan's
 * previous launch), and earl_plan_sync / earl_plan_destroy cover every launch. */
EARL_API earl_status_t earl_dispatch_exec(earl_plan_t plan, const void* const* send_bufs,
                                 void* const* recv_bufs, void* stream);
/* The fused dispatch of ONE source rank's records (data leaves "from their
 * computation origins"), to every destination replica it feeds; arguments as for
 * earl_dispatch_exec (only src_rank's send buffers are read).  Emulated comm: lets a source's
 * dispatch start as soon as its data is resident (e.g. overlapping the host-to-device copies of
 * the other sources); once every source rank has been executed, in any order, the recv buffers
 * equal those of one earl_dispatch_exec.  Multi-process comm: src_rank must be this rank (the
 * call is earl_dispatch_exec).  Launches of one plan share its scheduling counters: issue them
 * in one stream order, never concurrently.  Errors: INVALID_ARGUMENT for src_rank outside
 * [0, world) (or not this rank). */
EARL_API earl_status_t earl_dispatch_exec_src(earl_plan_t plan, int32_t src_rank,
                                              const void* const* send_bufs,
                                              void* const* recv_bufs, void* stream);
/* Staged path, step a3: gather this rank's segments into one contiguous message per
 * destination shard (field-major, each field block 16-byte aligned) in stage_bufs
 * ([1] or emulated [world]; size earl_plan_stats().stage_bytes[rank]).  send_bufs as for
 * earl_dispatch_exec (device, or mapped pinned host memory). */
EARL_API earl_status_t earl_dispatch_pack(earl_plan_t plan, const void* const* send_bufs,
                                 void* const* stage_bufs, void* stream);
/* Staged path, step a5: scatter packed messages into the final field arrays.
 * Emulated comm: stage_bufs [world] are the senders' stage buffers (as packed) and every
 *   destination replica's arrays are written (each message byte read once, written once per
 *   replica); recv_bufs is [world][n_fields].
 * Multi-process comm: stage_bufs[0] is this rank's receive buffer holding the messages it
 *   received, concatenated in source-rank order at the offsets earl_plan_messages reports;
 *   recv_bufs [n_fields] are this rank's field arrays. */
EARL_API earl_status_t earl_dispatch_unpack(earl_plan_t plan, const void* const* stage_bufs,
                                   void* const* recv_bufs, void* stream);

/* Staged path, step a4 bookkeeping for a multi-process exchange (e.g. grouped NCCL
 * send/recv): for rank `rank`, the byte range of its stage buffer to send to each peer d
 * (send_off[d], send_bytes[d]; message to d's shard, sent to every replica fed by this rank)
 * and where each source s's message lands in its receive buffer (recv_off[s], recv_bytes[s];
 * concatenated in source-rank order).  All arrays are HOST [world]; synchronises on the plan.
 * A rank's message to itself appears in both tables (copy it locally). */
EARL_API earl_status_t earl_plan_messages(earl_plan_t plan, int32_t rank, int64_t* send_off,
                                          int64_t* send_bytes, int64_t* recv_off,
                                          int64_t* recv_bytes);

/* ---- K8: the staged exchange over NCCL ------------------
 * The comparator of the fused P2P exec: pack -> grouped ncclSend / ncclRecv of the per-peer
 * messages (the earl_plan_messages table; a rank's message to itself goes through NCCL too) ->
 * unpack.  Two extra HBM passes and a host read of the byte table per call (NCCL takes host
 * sizes), against the fused exec's single pass; also the transport that crosses nodes. */

/* A fresh NCCL unique id (EARL_HANDLE_BYTES bytes) on one rank, to be broadcast out of band. */
EARL_API earl_status_t earl_nccl_unique_id(void* id_out);
/* Collective: create the comm's NCCL communicator (ncclCommInitRankConfig, world ranks, this
 * rank).  Knobs read here: EARL_NCCL_MIN_CTAS / EARL_NCCL_MAX_CTAS (config.minCTAs / maxCTAs),
 * EARL_NCCL_REGISTER=1 (stage buffers from ncclMemAlloc, registered with ncclCommRegister).
 * Errors: UNSUPPORTED (emulated comm), NCCL. */
EARL_API earl_status_t earl_comm_init_nccl(earl_comm_t comm, const void* unique_id);
/* Step a4 of the staged path: this rank's messages from send_stage (as earl_dispatch_pack left
 * them) to every peer, and every peer's message into recv_stage (concatenated in source-rank
 * order, the layout earl_dispatch_unpack reads), as one NCCL group on `stream`.  Synchronises
 * on the plan for the byte table.  Errors: INVALID_ARGUMENT (no NCCL comm, NULL stage with
 * bytes to move), NCCL. */
EARL_API earl_status_t earl_dispatch_exchange(earl_plan_t plan, const void* send_stage,
                                              void* recv_stage, void* stream);
/* pack + exchange + unpack with comm-owned stage buffers (grown on demand, outside the timed
 * steady state); send_bufs / recv_bufs as for earl_dispatch_exec (recv_bufs need not be in the
 * window).  Synchronises on the plan once per call. */
EARL_API earl_status_t earl_dispatch_exec_staged(earl_plan_t plan, const void* const* send_bufs,
                                                 void* const* recv_bufs, void* stream);

/* ---- NEXT-2: distributed aggregation before the dispatch ---------- */

/* On the source ranks (the plan's src layout must have sp == 1: sequences whole, as rollout DPn
 * holds them), per sequence, the discounted returns G_t = m_t r_t + gamma G_{t+1} (G_L = 0):
 * rewards fp32, mask u8 (1 = response token) and returns fp32 are this rank's token arrays
 * ([world] in an emulated comm), seq_return (optional, NULL) fp32 [n_local_seqs] gets G_0.
 * Accumulates the fp64 partials (sum m, sum m G, sum m G^2) of TP replica 0 into the DEVICE
 * array partial[3] (caller zeroes it).  Readings n5 in DESIGN.md.  Errors: UNSUPPORTED if the
 * source layout splits sequences (sp > 1).  Three kernels serve it, chosen by the
 * batch's size on the host, or on the device when the plan was re-planned since its last sync;
 * EARL_RETURNS=coop|units|windows forces one (a forced kernel the batch does not fit latches
 * CAPACITY, reported by the next synchronising call). */
EARL_API earl_status_t earl_returns(earl_plan_t plan, float gamma, const void* const* rewards,
                                    const void* const* mask, void* const* returns,
                                    void* const* seq_return, double* partial, void* stream);
/* A_t = m_t (G_t - mu) / (sigma + eps) with mu, sigma the mean and (population) standard
 * deviation of G over the batch's masked tokens, from stats[3] = the partials of earl_returns
 * summed over every rank (an all-reduce of 3 doubles in a multi-process comm: no controller
 * aggregates the rewards; REINFORCE++-style global normalisation). */
EARL_API earl_status_t earl_advantages(earl_plan_t plan, const double* stats, float eps,
                                       const void* const* returns, const void* const* mask,
                                       void* const* adv, void* stream);

/* ---- parallelism selector (host side of NEXT-4; Eq. (1))
 * "at the start of the training process, EARL measures the throughput under various
 * parallelism configurations and context lengths, then maintains the optimal configuration for
 * each context length range ... monitors the averaged context length ... When the averaged
 * context length falls into a new context range, EARL switches to the corresponding
 * parallelism configuration before the next Rollout stage."  Host-only: no CUDA calls, no
 * device memory.  The chosen configuration's layout is what the caller passes as `dst` (or
 * `src`) to earl_dispatch_plan.  Readings s1-s4 in DESIGN.md. */
typedef struct earl_policy* earl_policy_t;

/* Eq. (1): *out = (tgs_b - tgs_a) / tgs_a * 100 (positive: b is faster).
 * Errors: INVALID_ARGUMENT if tgs_a <= 0 or out is NULL. */
EARL_API earl_status_t earl_speedup_pct(double tgs_a, double tgs_b, double* out);

/* Build the selection table from a throughput profile.  n_configs configurations (config_tp[c] =
 * its TP degree, used only to break ties), n_buckets context ranges [bounds[b], bounds[b+1])
 * (bounds: n_buckets + 1 ascending token counts), tgs[c * n_buckets + b] = measured
 * tokens/GPU/s of configuration c in range b, oom[c * n_buckets + b] != 0 marks an OOM probe
 * (oom may be NULL).  Per range: the OOM-free configuration of highest TGS; ties go to the
 * smaller TP, then the lower index (s2).  hysteresis_tokens >= 0 (s3).  Host pointers, read
 * during the call only; *out is owned by the caller (earl_policy_destroy).
 * Errors: INVALID_ARGUMENT (counts <= 0, bounds not ascending, TGS <= 0 on an OOM-free entry,
 * NULL pointers), POLICY (a range where every configuration OOMs; earl_last_error names it). */
EARL_API earl_status_t earl_policy_build(int32_t n_configs, const int32_t* config_tp,
                                         int32_t n_buckets, const int64_t* bounds,
                                         const double* tgs, const uint8_t* oom,
                                         int64_t hysteresis_tokens, earl_policy_t* out);
/* config_of_bucket[n_buckets] <- the table. */
EARL_API earl_status_t earl_policy_table(earl_policy_t policy, int32_t* config_of_bucket);
/* The configuration for the next rollout given the observed average length (s3 hysteresis: keep
 * `current` while avg_len stays within hysteresis_tokens of a boundary shared with a range of
 * `current`, unless `current` is an OOM entry of the new range: the selection is never an OOM
 * configuration).  *next = the configuration, *switched = (next != current).
 * Errors: INVALID_ARGUMENT (current outside [0, n_configs), NULL), POLICY (avg_len outside
 * [bounds[0], bounds[n_buckets])). */
EARL_API earl_status_t earl_policy_select(earl_policy_t policy, double avg_len, int32_t current,
                                          int32_t* next, int32_t* switched);
EARL_API earl_status_t earl_policy_destroy(earl_policy_t policy);
/* The averaged context length of a planned batch, T / N (s4), from the plan's header
 * (synchronises with the planner like earl_plan_stats).  Errors: INVALID_ARGUMENT if N = 0. */
EARL_API earl_status_t earl_plan_mean_length(earl_plan_t plan, double* avg);

/* ---- misc -------------------------------------------------------------------------- */
EARL_API const char* earl_status_string(earl_status_t status);
EARL_API const char* earl_last_error(void);
EARL_API int32_t earl_abi_version(void);
/* Number of device kernels the library launched since load (bench evidence). */
EARL_API uint64_t earl_kernel_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* EARL_DISPATCH_H_ */
