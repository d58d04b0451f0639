// copy.cu -- the byte-moving kernels of the dispatcher (SURVEY.md §8(a) a3 pack, a5 unpack,
// a6 fused direct/P2P, a7 completion).
//
// All three modes run the same persistent kernel (one CTA per SM, 8 warps) over the plan's
// copy records.  The work of a launch is a record-major cost space (bytes + a fixed cost per
// (record, field) piece); warps take units of it -- first a static one, then further units
// from a plan-owned atomic counter -- so a 32K-token sequence next to hundreds of 100-token
// ones is split by cost, not by sequence, and stragglers are absorbed.  Bytes move through a
// per-warp TMA ring (cp.async.bulk global->shared, mbarrier complete_tx) and leave either by
// cp.async.bulk shared->global (source and destination congruent mod 16, local destination)
// or by 16-B warp stores (realigned in registers with funnel shifts when they are not
// congruent -- the 4-B id/fp32 fields and 1-B masks start at arbitrary token offsets -- and for
// destinations on a peer GPU).  Replicated destinations (TP, reading c2) are written from the
// same shared-memory stage: each source byte is read once.  No tensor cores: the path is pure
// data movement (HBM roofline).
#include "earl_internal.cuh"

namespace earl {

namespace {

constexpr unsigned kFull = 0xffffffffu;
// Work units: per_warp / 32 for large launches (the tail of the last unit is what
// a warp can be left with), at least min(192 KB, per_warp / 4) for mid-size ones (every claim
// costs a binary search over the records) and 4 stages.  Measured per_warp / 8 before: c5-lt
// 0.917 -> 0.953, c3 0.941 -> 0.956, C5 long-tail 64 MiB/rank 0.742 -> 0.80, small launches
// unchanged.
constexpr uint64_t kUnitsPerWarpLarge = 32;
constexpr uint64_t kUnitMidBytes = 192 * 1024;

__device__ __forceinline__ void st_v4(void* p, const uint4& v) {
  *reinterpret_cast<uint4*>(p) = v;
}
// NEXT-3: one 16-B store to a multicast address reaches every member of the team (NVSwitch
// replicates it); the payload is opaque, the .f32 vector form only moves the bits
__device__ __forceinline__ void multimem_st_v4(void* p, const uint4& v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p),
               "f"(__uint_as_float(v.x)), "f"(__uint_as_float(v.y)), "f"(__uint_as_float(v.z)),
               "f"(__uint_as_float(v.w))
               : "memory");
}

// 16 bytes starting at byte sh (1..15) of the 32-byte pair (A, B): S4 = sh/4 (a template
// parameter: the word selection is resolved at compile time, the loop below is instantiated per
// S4 instead of switching per 16 B) and bits = 8*(sh%4), warp-uniform.
template <int S4>
__device__ __forceinline__ uint4 realign(const uint4& A, const uint4& B, int bits) {
  const uint32_t w[8] = {A.x, A.y, A.z, A.w, B.x, B.y, B.z, B.w};
  return make_uint4(__funnelshift_r(w[S4], w[S4 + 1], bits), __funnelshift_r(w[S4 + 1], w[S4 + 2], bits),
                    __funnelshift_r(w[S4 + 2], w[S4 + 3], bits), __funnelshift_r(w[S4 + 3], w[S4 + 4], bits));
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Signal every peer of `peers` (bit p: rank p takes part; a multi-node comm's peers are its node's
// ranks) by storing `value` into slot `slot_base + me` of its pad, then wait until every such
// peer's slot in my pad holds at least `want`.  Lane p handles peer p.  Returns the mask of peers
// that timed out; *got (lane p) is the value peer p left in my pad.
__device__ unsigned signal_and_wait(uint64_t* my_pad, uint64_t* const* peer_pad, uint32_t peers, int me,
                                    int slot_base, uint64_t value, uint64_t want,
                                    uint64_t timeout_ns, uint64_t* got) {
  const int lane = threadIdx.x & 31;
  const bool mine = (peers >> lane & 1u) && lane != me;
  if (mine) st_release_sys(peer_pad[lane] + slot_base + me, value);
  unsigned missing = 0;
  uint64_t v = want;
  if (mine) {
    const uint64_t t0 = globaltimer();
    while ((v = ld_acquire_sys(my_pad + slot_base + lane)) < want) {
      if (globaltimer() - t0 > timeout_ns) { missing = 1u << lane; break; }
      __nanosleep(64);
    }
  }
  if (got) *got = v;
  return __reduce_or_sync(kFull, missing);
}

// The exec epoch lives in this rank's pad (slot kEpochSlot, written only by this rank): the
// entry barrier of every exec advances it and the copy kernel that follows on the stream reads
// it, so an exec captured into a CUDA graph gets a fresh epoch on every replay.
//
// Before signalling, this rank publishes where its receive buffers are (window offsets, one per
// field) in its own pad; after acquiring peer p's ready flag, lane p reads p's published offsets
// and resolves p's destination bases in this rank's address space (its mapping of p's window).
// Every rank therefore writes at the offsets the DESTINATION chose -- a rank that receives
// nothing (or is in no destination layout) may pass NULLs without silencing its own sends.
// Ordering: a peer reads these offsets only after acquiring this epoch's ready flag, and this
// rank rewrites them only in its next exec, after every peer released its done flag (i.e.
// finished reading).
__global__ void entry_barrier_kernel(uint64_t* my_pad, PeerPads pads, int world, uint32_t peers,
                                     int me, int n_fields, RecvOffsets offs, McTeams mct,
                                     uint64_t timeout_ns, int32_t* err, int32_t* err_detail) {
  const int lane = threadIdx.x & 31;
  uint64_t epoch = 0;
  if (lane == 0) {
    epoch = my_pad[kEpochSlot] + 1;
    my_pad[kEpochSlot] = epoch;
  }
  epoch = __shfl_sync(kFull, epoch, 0);
  if (lane < kMaxFields) my_pad[kOffSlot + lane] = lane < n_fields ? offs.v[lane] : kNoOffset;
  __threadfence_system();
  __syncwarp();
  delay_inject(1);
  const unsigned miss = signal_and_wait(my_pad, pads.p, peers, me, kReadySlot, epoch, epoch,
                                        timeout_ns, nullptr);
  // lane p: peer p's (or, for p == me, this rank's own) destination bases
  uint64_t* tab = my_pad + kDstTabSlot;
  if (lane < kMaxWorld) {
    for (int f = 0; f < kMaxFields; ++f) {
      uint64_t o = kNoOffset;
      if (lane < world && (lane == me || (peers >> lane & 1u)) && f < n_fields && !(miss >> lane & 1)) {
        o = lane == me ? offs.v[f]
                       : *reinterpret_cast<volatile const uint64_t*>(pads.p[lane] + kOffSlot + f);
      }
      tab[lane * kMaxFields + f] =
          o == kNoOffset ? 0ull : reinterpret_cast<uint64_t>(reinterpret_cast<uint8_t*>(pads.p[lane]) + o);
    }
  }
  if (lane == 0 && miss) {
    if (atomicCAS(err, 0, EARL_ERR_TIMEOUT) == 0) *err_detail = (int32_t)miss;
  }
  // NEXT-3: the multicast base of (dst shard ds, field f) when every member of ds's team put
  // field f at the same window offset (a multicast store lands at one offset on all of them)
  __syncwarp();
  __threadfence_block();
  uint64_t* mtab = my_pad + kMcTabSlot;
  if (lane < kMaxShards) {
    const int ds = lane;
    for (int f = 0; f < kMaxFields; ++f) {
      uint64_t v = 0;
      if (mct.va[ds] != 0 && f < n_fields && !miss) {
        uint64_t off = kNoOffset;
        bool same = true;
        for (int p = 0; p < world && same; ++p) {
          if (!(mct.mask[ds] >> p & 1)) continue;
          const uint64_t b = tab[p * kMaxFields + f];
          const uint64_t o = b ? b - reinterpret_cast<uint64_t>(pads.p[p]) : kNoOffset;
          if (o == kNoOffset || (off != kNoOffset && o != off)) same = false;
          off = o;
        }
        if (same && off != kNoOffset) v = mct.va[ds] + off;
      }
      mtab[ds * kMaxFields + f] = v;
    }
  }
}

// ---------------------------------------------------------------------------------------
// TMA-pipelined copy engine.  Each warp owns a ring of STAGES shared-memory buffers of CHUNK
// bytes.  Lane 0 walks the warp's byte slice (records x fields, cut into source-aligned
// chunks), writes a chunk descriptor and issues one cp.async.bulk global->shared per chunk
// (mbarrier complete_tx), STAGES-1 chunks ahead.  When a chunk lands, the warp stores it:
// if source and destination are congruent mod 16 the 16-B-aligned interior leaves shared
// memory by one cp.async.bulk shared->global per destination replica; otherwise all lanes
// realign it (two 16-B shared loads + funnel shift per 16-B output) into 16-B global stores.
// The <16-byte head and tail go byte by byte.  No data passes through registers on the
// congruent path, so the bytes in flight per SM are set by the ring, not by occupancy.
// ---------------------------------------------------------------------------------------

// One contiguous source range landed in a stage at stage offset `so` (a stage holds up to
// kSubs of them: small pieces share a stage, so the bytes in flight are set by the ring and
// not by the number of pieces).
struct __align__(16) SubDesc {
  const uint8_t* src_al;  // 16-B aligned source address of the load
  uint8_t* dst0;          // destination of the first byte for replica 0
  uint32_t so;            // stage offset of the load (multiple of 16)
  uint16_t load_bytes;    // multiple of 16 (<= CHUNK <= 16 KB)
  uint8_t rmask;          // replicas r < R that receive (a NULL receive buffer, another node)
  uint8_t pad_;
  uint32_t len;           // bytes
  uint8_t off;            // src & 15
  uint8_t R;              // destination replicas
  uint8_t f;              // field (replica base lookup)
  uint8_t d0;             // destination rank of replica 0 (direct / unpack)
};
static_assert(sizeof(SubDesc) == 32, "SubDesc layout");

constexpr int kSubs = 16;        // sub-ranges per stage
constexpr uint32_t kMinSpace = 256;  // close a stage when less than this is left

struct __align__(16) StageDesc {
  uint32_t n;
  uint32_t pad_[3];
  SubDesc sub[kSubs];
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store(void* gdst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_u32(smem_src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// The records a launch moves, as up to 8 contiguous blocks of the (s, ds, i, x)-ordered record
// table: everything (emulated comm), this rank's own records (fused exec / pack), or, for the
// unpack of a real rank, one block per source rank that sends to it -- each with the start of
// that source's message in this rank's receive buffer (messages concatenated in rank order).
struct View {
  int n;
  int64_t rbeg[kMaxWorld], rend[kMaxWorld], tbeg[kMaxWorld];
  uint64_t cbase[kMaxWorld + 1];
  const uint8_t* msg[kMaxWorld];
};

__device__ void build_view(const CopyArgs& a, uint64_t c0, View& v) {
  const PlanHeader* h = a.hdr;
  const int F = a.n_fields;
  const uint64_t B = a.Bpre[F];
  v.n = 0;
  v.cbase[0] = 0;
  auto add = [&](int64_t rb, int64_t re, const uint8_t* msg) {
    if (re <= rb) return;
    const int64_t t0 = a.rec.tok_prefix[rb], t1 = a.rec.tok_prefix[re];
    v.rbeg[v.n] = rb; v.rend[v.n] = re; v.tbeg[v.n] = t0; v.msg[v.n] = msg;
    v.cbase[v.n + 1] = v.cbase[v.n] + (uint64_t)(t1 - t0) * B + (uint64_t)(re - rb) * F * c0;
    ++v.n;
  };
  if (a.view_rank < 0) {
    add(0, h->n_records, nullptr);
  } else if (a.mode != kUnpack) {
    if (a.ds_mask == ~0u) {
      add(h->rec_begin[a.view_rank], h->rec_begin[a.view_rank + 1], nullptr);
    } else {  // NEXT-4: only the destination shards in ds_mask (messages that leave the node)
      const int Sd = a.n_dst_shards, r = a.view_rank;
      for (int ds = 0; ds < Sd; ++ds)
        if (a.ds_mask >> ds & 1u)
          add(h->rec_base[r][ds], ds + 1 < Sd ? h->rec_base[r][ds + 1] : h->rec_begin[r + 1], nullptr);
    }
  } else {
    const int Sd = a.n_dst_shards;
    const int rr = a.me - a.rank0_d;
    if (rr < 0 || rr >= Sd * a.tp_d) return;
    const int td = rr % a.tp_d, ds = rr / a.tp_d;
    const uint8_t* m = a.recv_stage;
    for (int s = 0; s < a.world; ++s) {
      const int q = s - a.rank0_s;
      if (q < 0 || q >= a.n_src_shards * a.tp_s) continue;
      const int ts = q % a.tp_s, ss = q / a.tp_s;
      if (ts >= a.nts || td % a.tp_s != ts) continue;
      if (!(a.src_mask >> s & 1u)) continue;  // NEXT-4: messages from other nodes only
      const int key = ss * Sd + ds;
      const int64_t rb = h->rec_base[s][ds];
      const int64_t re = (ds + 1 < Sd) ? h->rec_base[s][ds + 1] : h->rec_begin[s + 1];
      add(rb, re, m);
      for (int f = 0; f < F; ++f) m += (h->key_tokens[key] * a.Bf[f] + 15) & ~15LL;
    }
  }
}

// Lane-0-only walker over a warp's share of the launch's work.
//
// Work is measured in a record-major cost space: record j (all fields) of view block b
// occupies [cost(j), cost(j+1)) with cost(j) = cbase[b] + (tok_prefix[j] - tbeg[b]) * B +
// (j - rbeg[b]) * F * c0, and field f of record j is the sub-interval starting at
// n_j * Bpre[f] + f * c0 whose first n_j * B_f cost units map 1:1 to its bytes, followed by c0
// units that map to no bytes (the fixed cost of a piece).  Equal-byte slices made the warps
// holding thousands of small scalar pieces the stragglers; the c0 term balances them.
// Record-major order loads a record's metadata once for all of its fields.
//
// The walker holds scalars only (so it lives in registers); the launch's View (dynamically
// indexed, local memory) is consulted only when a warp changes block, and the kernel parameter
// is passed by reference into every (inlined) method so its fields are constant-bank loads.
struct Walker {
  int vn;  // the view's block count (a register copy; the View itself lives in local memory)
  int b;  // current view block and its fields
  int64_t b_rbeg, b_rend, b_tbeg;
  uint64_t b_cbase;
  const uint8_t* b_msg;
  uint64_t c0, x1, xpos, unit, n_units, first_dyn, total;
  // current record
  int64_t j;
  int f;
  uint64_t n, cj, fo;          // tokens, cost start, cost offset of field f inside the record
  int s, ds, ts, d0;
  int64_t src_tok, dst_tok, msg_tok, kt, msg_base, fb;
  // current piece (its own field and replica-0 rank: the walker may already have advanced)
  const uint8_t* psrc;
  uint8_t* pdst;
  uint32_t R, rmask;
  uint64_t prem;
  int pf, pd0;
  uint8_t* const* dt;  // the launch's destination field bases [kMaxWorld][kMaxFields] (smem)
  uint8_t* const* mt;  // NEXT-3: multicast bases [kMaxShards][kMaxFields] (smem), or nullptr

  __device__ __forceinline__ void set_block(const View& v, int bb) {
    b = bb;
    if (bb < vn) {
      b_rbeg = v.rbeg[bb]; b_rend = v.rend[bb]; b_tbeg = v.tbeg[bb]; b_cbase = v.cbase[bb];
      b_msg = v.msg[bb];
    } else {
      b_rbeg = b_rend = b_tbeg = 0; b_cbase = 0; b_msg = nullptr;
    }
  }

  __device__ __forceinline__ void setup(const CopyArgs& a, const View& v, uint64_t c0_,
                                        uint64_t first_dyn_) {
    vn = v.n;
    c0 = c0_; unit = 0; n_units = 0; first_dyn = first_dyn_; total = v.cbase[v.n];
    prem = 0; R = 0; xpos = x1 = 0; f = 0;
    set_block(v, 0);
    j = b_rbeg;
  }

  __device__ __forceinline__ uint64_t cost(const CopyArgs& a, int64_t jj) const {
    const int F = a.n_fields;
    return b_cbase + (uint64_t)(a.rec.tok_prefix[jj] - b_tbeg) * a.Bpre[F] +
           (uint64_t)(jj - b_rbeg) * F * c0;
  }

  __device__ __forceinline__ void load_record(const CopyArgs& a, int64_t jj) {
    const int F = a.n_fields;
    j = jj;
    const int64_t t0 = a.rec.tok_prefix[jj], t1 = a.rec.tok_prefix[jj + 1];
    const uint32_t code = a.rec.code[jj];
    src_tok = a.rec.src_tok[jj];
    dst_tok = a.rec.dst_tok[jj];
    n = (uint64_t)(t1 - t0);
    cj = b_cbase + (uint64_t)(t0 - b_tbeg) * a.Bpre[F] + (uint64_t)(jj - b_rbeg) * F * c0;
    s = code & 0xff;
    const int ss = (code >> 8) & 0xff;
    ds = (code >> 16) & 0xff;
    ts = code >> 24;
    d0 = a.rank0_d + ds * a.tp_d + ts;
    if (a.mode != kDirect) {
      const int key = ss * a.n_dst_shards + ds;
      msg_tok = a.rec.msg_tok[jj];
      kt = a.hdr->key_tokens[key];
      msg_base = a.hdr->msg_off[key];
    }
    f = 0;
    fo = 0;
    fb = 0;
  }

  __device__ __forceinline__ void next_field(const CopyArgs& a) {
    if (a.mode != kDirect) fb += (kt * a.Bf[f] + 15) & ~15LL;
    fo += n * a.Bf[f] + c0;
    ++f;
  }

  __device__ __forceinline__ void start(const CopyArgs& a, const View& v, uint64_t x0,
                                        uint64_t x1_) {
    x1 = x1_ < total ? x1_ : total;
    xpos = x0;
    prem = 0;
    if (xpos >= x1) return;
    int bb = 0;
    while (bb + 1 < vn && v.cbase[bb + 1] <= xpos) ++bb;
    set_block(v, bb);
    int64_t lo = b_rbeg, hi = b_rend - 1;  // last record whose cost starts <= xpos
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (cost(a, mid) <= xpos) lo = mid; else hi = mid - 1;
    }
    load_record(a, lo);
    while (f + 1 < a.n_fields && cj + fo + n * a.Bf[f] + c0 <= xpos) next_field(a);
  }

  // Position the walker at cost x0 with the whole warp (32-ary search; lane 0 holds the walker)
  __device__ __forceinline__ void start_warp(const CopyArgs& a, const View& v, uint64_t x0,
                                             uint64_t x1_, uint64_t c0w, int lane) {
    int64_t rb = 0, re = 0, tb = 0;
    uint64_t cb = 0;
    int go = 0;
    if (lane == 0) {
      x1 = x1_ < total ? x1_ : total;
      xpos = x0;
      prem = 0;
      if (xpos < x1) {
        int bb = 0;
        while (bb + 1 < vn && v.cbase[bb + 1] <= xpos) ++bb;
        set_block(v, bb);
        rb = b_rbeg; re = b_rend; tb = b_tbeg; cb = b_cbase;
        go = 1;
      }
    }
    if (!__shfl_sync(kFull, go, 0)) return;
    rb = __shfl_sync(kFull, rb, 0);
    re = __shfl_sync(kFull, re, 0);
    tb = __shfl_sync(kFull, tb, 0);
    cb = __shfl_sync(kFull, cb, 0);
    const int F = a.n_fields;
    const uint64_t B = a.Bpre[F];
    int64_t lo = rb, hi = re - 1;
    while (hi > lo) {
      const int64_t step = (hi - lo + 31) / 32;
      const int64_t pj = lo + (int64_t)lane * step;
      const bool ok = pj <= hi &&
                      cb + (uint64_t)(a.rec.tok_prefix[pj] - tb) * B + (uint64_t)(pj - rb) * F * c0w <= x0;
      const unsigned m = __ballot_sync(kFull, ok);
      const int l = 31 - __clz(m);
      lo = lo + (int64_t)l * step;
      hi = lo + step - 1 < hi ? lo + step - 1 : hi;
    }
    if (lane == 0) {
      load_record(a, lo);
      while (f + 1 < a.n_fields && cj + fo + n * a.Bf[f] + c0 <= xpos) next_field(a);
    }
  }

  // Claim the next unit: returns false when the launch's work is exhausted.
  __device__ __forceinline__ bool claim(const CopyArgs& a, const View& v) {
    const uint64_t u = first_dyn + atomicAdd(a.work_ctr, 1u);
    if (u >= n_units) return false;
    start(a, v, u * unit, (u + 1) * unit);
    return true;
  }

  __device__ __forceinline__ bool next_piece(const CopyArgs& a, const View& v) {
    const bool unpack_rank = a.mode == kUnpack && a.view_rank >= 0;
    while (xpos < x1) {
      const uint64_t Bf = a.Bf[f];
      const uint64_t nb = n * Bf;
      const uint64_t fstart = cj + fo, fend = fstart + nb + c0;
      const uint64_t lo = xpos - fstart;
      const uint64_t hi = (x1 < fend ? x1 : fend) - fstart;
      const uint64_t u0 = lo < nb ? lo : nb;
      const uint64_t u1 = hi < nb ? hi : nb;
      bool found = false;
      if (u1 > u0) {
        int64_t msg_field = 0;
        if (a.mode != kDirect) msg_field = msg_base + fb + msg_tok * (int64_t)Bf + (int64_t)u0;
        if (a.mode == kUnpack) {
          psrc = unpack_rank ? b_msg + fb + msg_tok * (int64_t)Bf + (int64_t)u0
                             : a.stage[s] + msg_field;
        } else {
          psrc = a.src[s][f] + src_tok * (int64_t)Bf + (int64_t)u0;
        }
        if (a.mode == kPack) {
          pdst = a.stage[s] + msg_field;
          R = 1;
          rmask = 1;
          pd0 = d0;
        } else if (unpack_rank) {
          uint8_t* base = dt[a.me * kMaxFields + f];
          pdst = base + dst_tok * (int64_t)Bf + (int64_t)u0;
          R = base != nullptr ? 1 : 0;
          rmask = 1;
          pd0 = a.me;
        } else {
          // replicas td = ts, ts + tp_s, ... of the shard; the ones with a receive buffer in
          // this launch (NULL: the rank receives nothing, or it is on another node) form rmask,
          // counted from the first present one
          uint32_t m = 0;
          int nrep = 0;
          for (int td = ts; td < a.tp_d; td += a.tp_s, ++nrep)
            if (dt[(d0 + (td - ts)) * kMaxFields + f] != nullptr) m |= 1u << nrep;
          R = 0;
          rmask = 0;
          pd0 = d0;
          if (m) {
            const int r0 = __ffs(m) - 1;
            rmask = m >> r0;
            R = 32 - __clz(rmask);
            pd0 = d0 + r0 * a.tp_s;
            pdst = dt[pd0 * kMaxFields + f] + dst_tok * (int64_t)Bf + (int64_t)u0;
          }
          // NEXT-3: every replica of this shard is in a multicast team with this rank
          if (mt != nullptr && R > 1 && rmask == (1u << R) - 1u && mt[ds * kMaxFields + f] != nullptr)
            R |= 0x80u;
        }
        prem = u1 - u0;
        pf = f;
        found = R > 0;
      }
      if (x1 >= fend) {
        xpos = fend;
        if (f + 1 < a.n_fields) {
          next_field(a);
        } else if (j + 1 < b_rend) {
          load_record(a, j + 1);
        } else if (b + 1 < vn) {
          set_block(v, b + 1);
          load_record(a, b_rbeg);
        } else {
          xpos = x1;
        }
      } else {
        xpos = x1;
      }
      if (found) return true;
    }
    return false;
  }

  // Next source range of at most `space` stage bytes (space >= kMinSpace): false when the
  // launch's work is exhausted.
  __device__ __forceinline__ bool next_sub(const CopyArgs& a, const View& v, SubDesc& d,
                                           uint32_t space) {
    while (prem == 0 && !next_piece(a, v))
      if (!claim(a, v)) return false;
    const uint32_t off = (uint32_t)((uintptr_t)psrc & 15);
    const uint64_t room = space - off;
    uint32_t len = (uint32_t)(prem < room ? prem : room);
    if (len < prem) {
      // more of this piece follows: end the range on a 128-B source boundary so the following
      // bulk copies cover whole cache lines
      const uint32_t cut = (uint32_t)(((uintptr_t)psrc + len) & 127);
      if (cut < len) len -= cut;
    }
    d.src_al = psrc - off;
    d.dst0 = pdst;
    d.off = (uint8_t)off;
    d.len = len;
    d.load_bytes = (uint16_t)((off + len + 15) & ~15u);
    d.R = (uint8_t)R;
    d.rmask = (uint8_t)rmask;
    d.f = (uint8_t)pf;
    d.d0 = (uint8_t)pd0;
    psrc += len;
    pdst += len;
    prem -= len;
    return true;
  }
};

// Fill stage `st` (lane 0): pack source ranges until the stage is full, then one expect_tx for
// the total and one TMA load per range, all completing on the stage's mbarrier.
template <int CHUNK>
__device__ __forceinline__ bool fill_stage(const CopyArgs& a, const View& v, Walker& wk,
                                           StageDesc& sd, uint8_t* stage, uint64_t* bar) {
  uint32_t used = 0, n = 0;
  while (n < (uint32_t)kSubs && CHUNK - used >= kMinSpace) {
    if (!wk.next_sub(a, v, sd.sub[n], CHUNK - used)) break;
    sd.sub[n].so = used;
    used += sd.sub[n].load_bytes;
    ++n;
  }
  sd.n = n;
  if (n == 0) return false;
  mbar_expect_tx(bar, used);
  for (uint32_t k = 0; k < n; ++k)
    tma_load(stage + sd.sub[k].so, sd.sub[k].src_al, sd.sub[k].load_bytes, bar);
  return true;
}

// The realigning warp-store loop of a non-congruent range: 16-B outputs k = lane, lane + 32, ...
// from the 32 bytes at sp + 16 (k - lane), one st.global.v4 per replica.
template <int R, int S4>
__device__ __forceinline__ void realign_loop(uint8_t* (&q)[R], const bool (&on)[R], const uint8_t* sp,
                                             uint32_t nvec, int bits, int lane) {
#pragma unroll 2
  for (uint32_t k = lane; k < nvec; k += 32) {
    const uint4 w0 = *reinterpret_cast<const uint4*>(sp);
    const uint4 w1 = *reinterpret_cast<const uint4*>(sp + 16);
    const uint4 o = realign<S4>(w0, w1, bits);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (on[r]) st_v4(q[r], o);
      q[r] += 512;
    }
    sp += 512;
  }
}

// Store one landed source range to its R destination replicas (whole warp); R is a
// compile-time constant so the replica pointers stay in registers and the realign loop is
// ~12 instructions per 512 B (a runtime-R loop cost ~100: profiles/r01_c5lt_note.txt).
// Replica r receives only if bit r of S.rmask is set (its rank passed a receive buffer and, in a
// multi-node comm, is on this node).
template <int R>
__device__ __forceinline__ void store_sub_r(const CopyArgs& a, uint8_t* const* dt, const SubDesc& S,
                                            uint8_t* stage, int lane) {
  const uint32_t len = S.len;
  const uint8_t* sm = stage + S.so + S.off;
  uint8_t* dp[R];
  bool on[R];
  dp[0] = S.dst0;
#pragma unroll
  for (int r = 0; r < R; ++r) on[r] = (S.rmask >> r) & 1u;
#pragma unroll
  for (int r = 1; r < R; ++r)
    dp[r] = S.dst0 + (dt[(S.d0 + r * a.tp_s) * kMaxFields + S.f] - dt[S.d0 * kMaxFields + S.f]);
  uint32_t head = (16 - (uint32_t)((uintptr_t)S.dst0 & 15)) & 15;
  if (head > len) head = len;
  if (lane < (int)head) {
    const uint8_t v = sm[lane];
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (on[r]) dp[r][lane] = v;
  }
  const uint32_t rest = len - head;
  const uint32_t nvec = rest >> 4;
  if (nvec > 0) {
    const uint32_t smo = S.so + S.off + head;
    if ((smo & 15) == 0) {
      // local replicas: one bulk TMA store each; replicas on a peer GPU (multi-process comm)
      // are written by the warp with 16-B stores over NVLink, or (EARL_REMOTE_STORE=tma) by
      // bulk TMA stores to the peer address as well
      bool remote[R];
      bool any_remote = false;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        remote[r] = on[r] && !a.remote_tma && a.mode != kPack && a.me >= 0 && (S.d0 + r * a.tp_s) != a.me;
        any_remote |= remote[r];
      }
      if (lane == 0) {
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (on[r] && !remote[r]) tma_store(dp[r] + head, stage + smo, nvec * 16);
      }
      if (any_remote) {
        for (uint32_t k = lane; k < nvec; k += 32) {
          const uint4 v = *reinterpret_cast<const uint4*>(stage + smo + 16 * k);
#pragma unroll
          for (int r = 0; r < R; ++r)
            if (remote[r]) st_v4(dp[r] + head + 16 * k, v);
        }
      }
    } else {
      const uint32_t sh = smo & 15;
      const int bits = (int)(sh & 3) * 8;
      const uint8_t* sp = stage + (smo & ~15u) + 16 * lane;
      uint8_t* q[R];
#pragma unroll
      for (int r = 0; r < R; ++r) q[r] = dp[r] + head + 16 * lane;
      switch (sh >> 2) {
        case 0: realign_loop<R, 0>(q, on, sp, nvec, bits, lane); break;
        case 1: realign_loop<R, 1>(q, on, sp, nvec, bits, lane); break;
        case 2: realign_loop<R, 2>(q, on, sp, nvec, bits, lane); break;
        default: realign_loop<R, 3>(q, on, sp, nvec, bits, lane); break;
      }
    }
  }
  const uint32_t t0 = head + nvec * 16;
  if (lane < (int)(len - t0)) {
    const uint8_t v = sm[t0 + lane];
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (on[r]) dp[r][t0 + lane] = v;
  }
}

// NEXT-3: a range whose R replicas form a multicast team this rank belongs to: the 16-B interior
// leaves once, by multimem.st to the team's address (reaching every replica, this rank's own
// included); heads and tails (< 16 B each) go byte by byte to every replica.
template <int R>
__device__ __forceinline__ void store_sub_mc(const CopyArgs& a, uint8_t* const* dt,
                                             uint8_t* const* mt, const SubDesc& S, uint8_t* stage,
                                             int lane) {
  const uint32_t len = S.len;
  const uint8_t* sm = stage + S.so + S.off;
  uint8_t* dp[R];
  dp[0] = S.dst0;
#pragma unroll
  for (int r = 1; r < R; ++r)
    dp[r] = S.dst0 + (dt[(S.d0 + r * a.tp_s) * kMaxFields + S.f] - dt[S.d0 * kMaxFields + S.f]);
  const int ds = (S.d0 - a.rank0_d) / a.tp_d;
  uint8_t* mc = mt[ds * kMaxFields + S.f] + (S.dst0 - dt[S.d0 * kMaxFields + S.f]);
  uint32_t head = (16 - (uint32_t)((uintptr_t)S.dst0 & 15)) & 15;
  if (head > len) head = len;
  if (lane < (int)head) {
    const uint8_t v = sm[lane];
#pragma unroll
    for (int r = 0; r < R; ++r) dp[r][lane] = v;
  }
  const uint32_t rest = len - head;
  const uint32_t nvec = rest >> 4;
  if (nvec > 0) {
    const uint32_t smo = S.so + S.off + head;
    const uint32_t sh = smo & 15;
    const uint8_t* sp = stage + (smo & ~15u);
    for (uint32_t k = lane; k < nvec; k += 32) {
      uint4 o;
      const uint4 w0 = *reinterpret_cast<const uint4*>(sp + 16 * k);
      if (sh == 0) {
        o = w0;
      } else {
        const uint4 w1 = *reinterpret_cast<const uint4*>(sp + 16 * k + 16);
        const int bits = (int)(sh & 3) * 8;
        switch (sh >> 2) {
          case 0: o = realign<0>(w0, w1, bits); break;
          case 1: o = realign<1>(w0, w1, bits); break;
          case 2: o = realign<2>(w0, w1, bits); break;
          default: o = realign<3>(w0, w1, bits); break;
        }
      }
      multimem_st_v4(mc + head + 16 * k, o);
    }
  }
  const uint32_t t0 = head + nvec * 16;
  if (lane < (int)(len - t0)) {
    const uint8_t v = sm[t0 + lane];
#pragma unroll
    for (int r = 0; r < R; ++r) dp[r][t0 + lane] = v;
  }
}

__device__ __forceinline__ void store_sub_mc_any(const CopyArgs& a, uint8_t* const* dt,
                                                 uint8_t* const* mt, const SubDesc& S,
                                                 uint8_t* stage, int lane) {
  switch (S.R & 0x7f) {
    case 2: store_sub_mc<2>(a, dt, mt, S, stage, lane); break;
    case 3: store_sub_mc<3>(a, dt, mt, S, stage, lane); break;
    case 4: store_sub_mc<4>(a, dt, mt, S, stage, lane); break;
    case 5: store_sub_mc<5>(a, dt, mt, S, stage, lane); break;
    case 6: store_sub_mc<6>(a, dt, mt, S, stage, lane); break;
    case 7: store_sub_mc<7>(a, dt, mt, S, stage, lane); break;
    default: store_sub_mc<8>(a, dt, mt, S, stage, lane); break;
  }
}

__device__ __forceinline__ void store_sub(const CopyArgs& a, uint8_t* const* dt, const SubDesc& S,
                                          uint8_t* stage, int lane) {
  switch (S.R) {
    case 1: store_sub_r<1>(a, dt, S, stage, lane); break;
    case 2: store_sub_r<2>(a, dt, S, stage, lane); break;
    case 3: store_sub_r<3>(a, dt, S, stage, lane); break;
    case 4: store_sub_r<4>(a, dt, S, stage, lane); break;
    case 5: store_sub_r<5>(a, dt, S, stage, lane); break;
    case 6: store_sub_r<6>(a, dt, S, stage, lane); break;
    case 7: store_sub_r<7>(a, dt, S, stage, lane); break;
    default: store_sub_r<8>(a, dt, S, stage, lane); break;
  }
}

template <int WARPS, int STAGES, int CHUNK>
constexpr size_t copy_smem_bytes() {
  return (size_t)WARPS * STAGES * CHUNK + (size_t)WARPS * STAGES * (sizeof(StageDesc) + 8);
}

template <int WARPS, int STAGES, int CHUNK, bool MC>
__global__ void __launch_bounds__(WARPS * 32, 1) copy_kernel(const __grid_constant__ CopyArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ unsigned s_last;
  __shared__ uint8_t* s_dst[kMaxWorld * kMaxFields];
  __shared__ uint8_t* s_mc[MC ? kMaxShards * kMaxFields : 1];  // NEXT-3: multicast bases
  if (MC)
    for (int k = threadIdx.x; k < kMaxShards * kMaxFields; k += WARPS * 32) s_mc[k] = a.mc_tab[k];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // destination field bases: the kernel parameter, or (multi-process exec) the table the entry
  // barrier resolved from every destination's published offsets
  for (int k = threadIdx.x; k < kMaxWorld * kMaxFields; k += WARPS * 32)
    s_dst[k] = a.protocol ? a.dst_tab[k] : a.dst[k / kMaxFields][k % kMaxFields];
  uint8_t* data = smem + (size_t)w * STAGES * CHUNK;
  StageDesc* desc = reinterpret_cast<StageDesc*>(smem + (size_t)WARPS * STAGES * CHUNK) + w * STAGES;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + (size_t)WARPS * STAGES * CHUNK +
                                              (size_t)WARPS * STAGES * sizeof(StageDesc)) + w * STAGES;
  if (lane == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  delay_inject(2);
  const PlanHeader* h = a.hdr;
  if (h->err == 0) {
    const uint64_t c0 = CHUNK / 4;
    const uint64_t nwarps = (uint64_t)gridDim.x * WARPS;
    const uint64_t wid = (uint64_t)blockIdx.x * WARPS + w;
    Walker wk;
    View v;
    uint64_t t_start = 0;
    int nprod = 0;
    if (lane == 0) {
      if (a.trace) t_start = globaltimer();
      build_view(a, c0, v);
      wk.setup(a, v, c0, nwarps);
      wk.dt = s_dst;
      wk.mt = MC ? s_mc : nullptr;
      const uint64_t total = wk.total;
      // units: every warp starts on unit `wid`, then claims units >= nwarps dynamically
      const uint64_t per_warp = (total + nwarps - 1) / nwarps;
      const uint64_t mid = per_warp / 4 < kUnitMidBytes ? per_warp / 4 : kUnitMidBytes;
      uint64_t unit = (per_warp + kUnitsPerWarpLarge - 1) / kUnitsPerWarpLarge;
      if (unit < mid) unit = mid;
      if (unit < 4 * (uint64_t)CHUNK) unit = 4 * (uint64_t)CHUNK;
      wk.unit = unit;
      wk.n_units = (total + unit - 1) / unit;
    }
    {
      const uint64_t nu = __shfl_sync(kFull, lane == 0 ? wk.n_units : 0ull, 0);
      const uint64_t un = __shfl_sync(kFull, lane == 0 ? wk.unit : 0ull, 0);
      if (wid < nu) wk.start_warp(a, v, wid * un, (wid + 1) * un, c0, lane);
    }
    for (int s = 0; s < STAGES - 1; ++s) {
      int ok = 0;
      if (lane == 0) ok = fill_stage<CHUNK>(a, v, wk, desc[s], data + (size_t)s * CHUNK, &bar[s]);
      ok = __shfl_sync(kFull, ok, 0);
      if (!ok) break;
      ++nprod;
    }
    for (int c = 0; c < nprod; ++c) {
      const int st = c % STAGES;
      mbar_wait(&bar[st], (uint32_t)((c / STAGES) & 1));
      uint8_t* stage = data + (size_t)st * CHUNK;
      const uint32_t nsub = desc[st].n;
      for (uint32_t k = 0; k < nsub; ++k) {
        if (MC && (desc[st].sub[k].R & 0x80))
          store_sub_mc_any(a, s_dst, s_mc, desc[st].sub[k], stage, lane);
        else
          store_sub(a, s_dst, desc[st].sub[k], stage, lane);
      }
      if (lane == 0) { bulk_commit(); bulk_wait_read1(); }
      __syncwarp();
      int ok = 0;
      if (lane == 0) {
        const int ns = (c + STAGES - 1) % STAGES;
        fence_proxy_async_smem();
        ok = fill_stage<CHUNK>(a, v, wk, desc[ns], data + (size_t)ns * CHUNK, &bar[ns]);
      }
      ok = __shfl_sync(kFull, ok, 0);
      if (ok) ++nprod;
    }
    if (lane == 0) bulk_wait_all();
    if (lane == 0 && a.trace) {
      uint64_t* t = a.trace + 4 * wid;
      t[0] = t_start; t[1] = globaltimer(); t[2] = wk.unit; t[3] = (uint64_t)nprod;
    }
    __syncwarp();
  }
  // the last CTA to finish resets the plan's scheduling counters for the next launch
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(a.fin_ctr, 1u) == gridDim.x - 1) {
      *a.work_ctr = 0;
      *a.fin_ctr = 0;
      __threadfence();
    }
  }
  // completion (multi-process comm): last CTA releases this epoch to every peer and waits
  if (a.protocol) {
    delay_inject(3);
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned prev = atomicAdd(a.done_ctr, 1u);
      s_last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (s_last && threadIdx.x < 32) {
      if (threadIdx.x == 0) *a.done_ctr = 0;
      __threadfence_system();
      // done = 2 * epoch + failed: a rank whose copies were skipped (its entry barrier timed out,
      // or its plan latched an error) says so, and every peer latches an error instead of
      // returning with that rank's contribution missing
      const uint64_t epoch = *reinterpret_cast<volatile uint64_t*>(a.my_pad + kEpochSlot);
      const uint64_t failed = *reinterpret_cast<volatile const int32_t*>(a.err) != 0 ? 1 : 0;
      uint64_t got = 0;
      const unsigned miss = signal_and_wait(a.my_pad, a.peer_pad, a.peer_mask, a.me, kDoneSlot,
                                            2 * epoch + failed, 2 * epoch, a.timeout_ns, &got);
      const int lane = threadIdx.x;
      const unsigned bad = __ballot_sync(kFull, (a.peer_mask >> lane & 1u) && lane != a.me &&
                                                    !(miss >> lane & 1) && got == 2 * epoch + 1);
      if (lane == 0 && (miss | bad)) {
        if (atomicCAS(a.err, 0, EARL_ERR_TIMEOUT) == 0) *a.err_detail = (int32_t)(miss | bad << 8);
      }
    }
  }
}

template <int WARPS, int STAGES, int CHUNK, bool MC = false>
cudaError_t launch_cfg(const CopyArgs& a, int sm_count, cudaStream_t s) {
  constexpr size_t smem = copy_smem_bytes<WARPS, STAGES, CHUNK>();
  static bool configured[64] = {};
  auto kern = copy_kernel<WARPS, STAGES, CHUNK, MC>;
  cudaError_t e = opt_in_dynamic_smem(kern, (int)smem, configured);
  if (e != cudaSuccess) return e;
  // resident CTAs per SM of this shape, queried once per device (a host call per launch showed
  // up in the small-batch step time)
  static int per_sm_of[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  int per_sm = dev >= 0 && dev < 64 ? per_sm_of[dev] : 0;
  if (per_sm <= 0) {
    per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WARPS * 32, smem);
    if (per_sm < 1) per_sm = 1;
    if (dev >= 0 && dev < 64) per_sm_of[dev] = per_sm;
  }
  kern<<<sm_count * per_sm, WARPS * 32, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

// Copy-engine shape (warps per CTA, ring stages, chunk bytes), chosen per launch from the field
// widths (measured): when nearly all bytes sit in fields whose width is a
// multiple of 16 B (hidden vectors: source and destination always congruent, bytes leave by TMA
// bulk stores) few warps with large stages win on TP-replicated stores: 2 warps x 2 stages x
// 16 KB (3 CTAs per SM) 0.933-0.940 of peak on c3 against 0.920 for 4 warps x 4 x 8 KB (1 CTA)
// on the same box, c4 1.00, c2-lpt 0.99; otherwise the realign path needs the issue slots of 8
// warps (0.93 vs 0.63 on the long-tail scalar sweep).  EARL_COPY_CFG forces a shape for tuning.
// shape >= 100: the shape id shape - 100, forced by the caller (multi-process P2P override).
cudaError_t launch_copy(const CopyArgs& a, int sm_count, int shape, cudaStream_t s) {
  static int forced = -2;
  if (forced == -2) {
    const char* e = getenv("EARL_COPY_CFG");
    forced = e ? atoi(e) : -1;
  }
  const int cfg = shape >= 100 ? shape - 100 : forced >= 0 ? forced : (shape ? 14 : 3);
  if (a.mc_on)  // NEXT-3: the multicast-capable instantiations of the two default shapes
    return cfg == 14 ? launch_cfg<2, 2, 16384, true>(a, sm_count, s) : launch_cfg<8, 3, 8192, true>(a, sm_count, s);
  switch (cfg) {
    case 1: return launch_cfg<8, 4, 4096>(a, sm_count, s);
    case 2: return launch_cfg<4, 4, 8192>(a, sm_count, s);
    case 4: return launch_cfg<2, 8, 8192>(a, sm_count, s);
    case 5: return launch_cfg<16, 2, 4096>(a, sm_count, s);
    case 6: return launch_cfg<8, 4, 6144>(a, sm_count, s);
    case 7: return launch_cfg<4, 3, 16384>(a, sm_count, s);
    case 8: return launch_cfg<2, 6, 16384>(a, sm_count, s);
    case 11: return launch_cfg<2, 4, 8192>(a, sm_count, s);
    case 14: return launch_cfg<2, 2, 16384>(a, sm_count, s);
    default: return launch_cfg<8, 3, 8192>(a, sm_count, s);
  }
}

cudaError_t launch_entry_barrier(uint64_t* my_pad, uint64_t* const* peer_pad, int world,
                                 uint32_t peers, int me, int n_fields, const uint64_t* recv_off,
                                 const McTeams& mct, uint64_t timeout_ns, int32_t* err,
                                 int32_t* err_detail, cudaStream_t s) {
  PeerPads pads;
  for (int p = 0; p < kMaxWorld; ++p) pads.p[p] = peer_pad[p];
  RecvOffsets offs;
  for (int f = 0; f < kMaxFields; ++f) offs.v[f] = f < n_fields ? recv_off[f] : kNoOffset;
  entry_barrier_kernel<<<1, 32, 0, s>>>(my_pad, pads, world, peers, me, n_fields, offs, mct,
                                        timeout_ns, err, err_detail);
  return cudaGetLastError();
}

}  // namespace earl
