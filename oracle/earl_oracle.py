"""CPU oracle for EARL's layout-aware decentralized data dispatch (arXiv 2510.05943).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import or execute anything under oracle/.
The product path (paper_2510_05943_b200 + its CUDA library) never imports this module,
and this module imports nothing from the product path.

What it computes (§2 "Data Dispatcher"): intermediate RL batches
(per-token fields of variable-length sequences) held by the
workers of one parallel layout are re-distributed to the workers of another layout
by sending "data directly to the target workers from their computation origins"
(PAPER.md:195), an all-to-all that replaces "all-gather-and-scatter".
The result is fully determined by the two layouts, so the oracle writes out the
plain definition, step by step, in the order of SURVEY.md §8(c):

  1 validate            -> validate_layout
  2 sequence identity   -> (index into seq_lens)
  3 assignment g(i)     -> assign_groups (GIVEN_COUNTS / CONTIG / LPT / EXPLICIT)
  4 SP chunking         -> sp_chunk (BLOCK rule, SPEC.md:215 remainder rule on tokens)
  5 holdings            -> holdings / rank_arrays_from_global
  6 routing             -> route (canonical order (s, d, i, x))
  7 messages            -> build_messages
  8 assembly            -> assemble
  9 brute force         -> brute_force (centralized gather-then-scatter)
 10 stats               -> stats

Plus the centralized gather-and-dispatch baseline of PAPER.md:163/194 as two dispatches
through one controller rank: gather_scatter_layouts.

Readings where the paper is silent are SURVEY.md §8(c) c1-c21 and are listed in DESIGN.md.
Everything is integer / byte work: payload bytes are opaque (reading c10) and are never
interpreted, so parity is bit-exact.

Pins (tests/test_oracle_*.py): hand-worked tiny case (tests/golden/c1_tiny.json),
SPEC.md worked examples, closed forms (textbook scan), LPT against exhaustive search,
an independently written per-token brute force, and the invariants exactly-once /
conservation / round-trip / dominance / determinism.
"""
from __future__ import annotations

import hashlib
import itertools

import numpy as np

# Status names mirror include/earl_dispatch.h's earl_status_t (the names only; no code is shared).
ERR_INVALID_ARGUMENT = "INVALID_ARGUMENT"
ERR_LAYOUT = "LAYOUT"
ERR_CAPACITY = "CAPACITY"
ERR_UNSUPPORTED = "UNSUPPORTED"

LPT_MAX_SEQS = 8192       # reading c4 / §8(b): LPT limited to N <= 8192
SP_SPLITS = ("block", "zigzag", "flat", "threshold")  # readings c7, n1-n3
MAX_WORLD = 8             # reading c21: one box, W <= 8
INT32_MAX = 2**31 - 1


class OracleError(Exception):
    def __init__(self, code, msg):
        super().__init__(f"{code}: {msg}")
        self.code = code


# ---------------------------------------------------------------------------
# layouts
# ---------------------------------------------------------------------------

def n_ranks(lay) -> int:
    return lay["dp"] * lay["sp"] * lay["tp"]


def rank_of(lay, g, k, t) -> int:
    """Reading c3: TP fastest, then SP, then DP: rank = rank0 + (g*SP + k)*TP + t."""
    return lay["rank0"] + (g * lay["sp"] + k) * lay["tp"] + t


def coords_of(lay, rank):
    """Inverse of rank_of; None if rank is not in the layout."""
    r = rank - lay["rank0"]
    if r < 0 or r >= n_ranks(lay):
        return None
    t = r % lay["tp"]
    gk = r // lay["tp"]
    return gk // lay["sp"], gk % lay["sp"], t


def validate_layout(lay, n_seqs, world):
    """Step 1 (SPEC.md:225 'coverage mismatch -> layout error'; §8(b) error list)."""
    if world < 1 or world > MAX_WORLD:
        raise OracleError(ERR_UNSUPPORTED, f"world {world} not in [1, {MAX_WORLD}]")
    if n_seqs < 0:
        raise OracleError(ERR_INVALID_ARGUMENT, "n_seqs < 0")
    for key in ("dp", "sp", "tp"):
        if lay[key] < 1:
            raise OracleError(ERR_LAYOUT, f"{key} < 1")
    if lay["rank0"] < 0 or lay["rank0"] + n_ranks(lay) > world:
        raise OracleError(ERR_LAYOUT, "layout ranks outside the comm")
    split = lay.get("sp_split", "block")
    if split not in SP_SPLITS:
        raise OracleError(ERR_INVALID_ARGUMENT, f"unknown sp_split {split!r}")
    if split == "threshold" and int(lay.get("sp_min_len", 0)) < 0:
        raise OracleError(ERR_INVALID_ARGUMENT, "sp_min_len < 0")
    a = lay["assign"]
    if a == "given_counts":
        c = lay["counts"]
        if c is None or len(c) != lay["dp"] or any(x < 0 for x in c) or sum(c) != n_seqs:
            raise OracleError(ERR_LAYOUT, "GIVEN_COUNTS must be dp non-negative counts summing to N")
    elif a == "explicit":
        gos = lay["group_of_seq"]
        if gos is None or len(gos) != n_seqs:
            raise OracleError(ERR_INVALID_ARGUMENT, "EXPLICIT needs group_of_seq[N]")
        for g in gos:
            if g < 0 or g >= lay["dp"]:
                raise OracleError(ERR_LAYOUT, "EXPLICIT group out of range")
    elif a == "lpt":
        if n_seqs > LPT_MAX_SEQS:
            raise OracleError(ERR_CAPACITY, f"LPT needs N <= {LPT_MAX_SEQS}")
    elif a != "contig":
        raise OracleError(ERR_INVALID_ARGUMENT, f"unknown assignment {a!r}")


def validate_lengths(seq_lens):
    """Reading c20: L_i < 0 is an invalid argument; L_i = 0 is valid."""
    for x in seq_lens:
        if int(x) < 0:
            raise OracleError(ERR_INVALID_ARGUMENT, "negative sequence length")


# ---------------------------------------------------------------------------
# step 3: assignment
# ---------------------------------------------------------------------------

def exclusive_scan(seq_lens):
    """P_i = sum_{j<i} L_j (int64) and T = sum L (SURVEY.md §8 notation)."""
    P = []
    acc = 0
    for x in seq_lens:
        P.append(acc)
        acc += int(x)
    return P, acc


def count_blocks(n, d):
    """Near-equal contiguous blocks, earlier groups get the extra (SPEC.md:212-220 block_layout)."""
    q, r = divmod(n, d)
    return [q + (1 if g < r else 0) for g in range(d)]


def groups_from_counts(counts):
    g_of = []
    for g, c in enumerate(counts):
        g_of.extend([g] * c)
    return g_of


def assign_contig(seq_lens, D):
    """CONTIG midpoint rule (reading c4): g(i) = min(D-1, floor(D*(2*P_i + L_i) / (2*T))).

    If T == 0, fall back to count blocks.
    """
    P, T = exclusive_scan(seq_lens)
    N = len(seq_lens)
    if T == 0:
        return groups_from_counts(count_blocks(N, D))
    return [min(D - 1, (D * (2 * P[i] + int(seq_lens[i]))) // (2 * T)) for i in range(N)]


def assign_lpt(seq_lens, D):
    """LPT (Graham's greedy), reading c4: visit i in order (L_i desc, i asc); put each into
    the group with the minimum current load, ties to the lowest group index."""
    order = sorted(range(len(seq_lens)), key=lambda i: (-int(seq_lens[i]), i))
    loads = [0] * D
    g_of = [0] * len(seq_lens)
    for i in order:
        best = 0
        for g in range(1, D):
            if loads[g] < loads[best]:
                best = g
        g_of[i] = best
        loads[best] += int(seq_lens[i])
    return g_of


def assign_groups(lay, seq_lens):
    """Step 3: g(i) for every sequence under the layout's assignment rule."""
    a, D = lay["assign"], lay["dp"]
    if a == "given_counts":
        return groups_from_counts(lay["counts"])
    if a == "contig":
        return assign_contig(seq_lens, D)
    if a == "lpt":
        return assign_lpt(seq_lens, D)
    if a == "explicit":
        return [int(g) for g in lay["group_of_seq"]]
    raise OracleError(ERR_INVALID_ARGUMENT, a)


# ---------------------------------------------------------------------------
# step 4: SP chunking
# ---------------------------------------------------------------------------

def sp_chunk(L, SP, k):
    """BLOCK rule (reading c7): q = L // SP, r = L % SP; chunk k = [k*q + min(k,r), (k+1)*q + min(k+1,r))."""
    q, r = divmod(int(L), SP)
    return k * q + min(k, r), (k + 1) * q + min(k + 1, r)


def group_members(seq_lens, g_of, D):
    """Sequences of every group in ascending global index (reading c5)."""
    members = {g: [] for g in range(D)}
    for i in range(len(seq_lens)):
        members[g_of[i]].append(i)
    return members


def seq_chunks(lay, seq_lens, g_of):
    """Step 4, generalised SP split.  For every sequence i, the ordered list of its virtual
    chunks (c, lo, hi, k): token range [lo, hi) of sequence i, held by SP rank k of its group.
    The chunks of a sequence are consecutive and cover [0, L_i).

      block     (reading c7)  c = k = 0..SP-1, chunk k = sp_chunk(L, SP, k)
      zigzag    (reading n1)  c = 0..2SP-1, chunk c = sp_chunk(L, 2SP, c), held by
                              k = c if c < SP else 2SP-1-c  (rank k holds chunks k and 2SP-1-k)
      flat      (reading n2)  the group's sequences concatenated in ascending i form a stream of
                              S_g tokens; SP rank k holds stream block sp_chunk(S_g, SP, k);
                              chunk k of sequence i is that block's intersection with i
      threshold (reading n3)  L >= sp_min_len: block; otherwise the whole sequence goes to SP
                              rank (position of i in its group) mod SP: chunk c = [0,0) before
                              that rank, [0,L) at it, [L,L) after it
    """
    SP = lay["sp"]
    split = lay.get("sp_split", "block")
    thresh = int(lay.get("sp_min_len", 0))
    out = {}
    for g, members in group_members(seq_lens, g_of, lay["dp"]).items():
        if split == "flat":
            S = sum(int(seq_lens[i]) for i in members)
            blocks = [sp_chunk(S, SP, k) for k in range(SP)]
            pos = 0
            for i in members:
                L = int(seq_lens[i])
                out[i] = [(k, min(max(a - pos, 0), L), min(max(b - pos, 0), L), k)
                          for k, (a, b) in enumerate(blocks)]
                pos += L
            continue
        for p, i in enumerate(members):
            L = int(seq_lens[i])
            if split == "zigzag":
                out[i] = [(c,) + sp_chunk(L, 2 * SP, c) + (c if c < SP else 2 * SP - 1 - c,)
                          for c in range(2 * SP)]
            elif split == "threshold" and L < thresh:
                owner = p % SP
                out[i] = [(c, 0 if c <= owner else L, 0 if c < owner else L, c) for c in range(SP)]
            else:
                out[i] = [(k,) + sp_chunk(L, SP, k) + (k,) for k in range(SP)]
    return out


# ---------------------------------------------------------------------------
# step 5: holdings
# ---------------------------------------------------------------------------

def holdings(lay, seq_lens, g_of):
    """Step 5: every rank (g, k, t) of the layout holds, for each sequence of group g in
    ascending i (reading c5), the chunks of that sequence SP rank k holds, in chunk order --
    i.e. its tokens in ascending position.  Also cu_seqlens (tokens held per sequence, scanned),
    seq_ids, tok_start (first token of the first held chunk) and each chunk's local offset.

    Returns dict rank -> {"chunks": [(i, c, lo, hi)], "local_off": {(i, c): offset},
    "cu_seqlens": [...], "seq_ids": [...], "tok_start": [...], "n_tokens": int}.
    """
    chunks_of = seq_chunks(lay, seq_lens, g_of)
    out = {}
    for g, members in group_members(seq_lens, g_of, lay["dp"]).items():
        for k in range(lay["sp"]):
            held = []
            local_off = {}
            cu = [0]
            tok_start = []
            for i in members:
                mine = [(c, lo, hi) for (c, lo, hi, kk) in chunks_of[i] if kk == k]
                tok_start.append(mine[0][1])
                total = cu[-1]
                for (c, lo, hi) in mine:
                    local_off[(i, c)] = total
                    held.append((i, c, lo, hi))
                    total += hi - lo
                cu.append(total)
            for t in range(lay["tp"]):
                out[rank_of(lay, g, k, t)] = {
                    "chunks": held,
                    "local_off": local_off,
                    "cu_seqlens": list(cu),
                    "seq_ids": list(members),
                    "tok_start": list(tok_start),
                    "n_tokens": cu[-1],
                }
    return out


def field_bytes(fields):
    """B_f = bytes_per_elem * elems_per_token for every field (§8 notation)."""
    return [int(f[1]) * int(f[2]) for f in fields]


def rank_arrays_from_global(lay, seq_lens, g_of, global_fields, fields):
    """The arrays every rank of `lay` holds, cut out of the global (sequence-order) arrays.

    Used to (a) build src holdings for tests and (b) as the 'scatter' half of the brute force.
    rank -> [per-field uint8 array of n_tokens*B_f bytes].
    """
    P, _ = exclusive_scan(seq_lens)
    Bf = field_bytes(fields)
    hold = holdings(lay, seq_lens, g_of)
    out = {}
    for r, h in hold.items():
        per_field = []
        for f, arr in enumerate(global_fields):
            parts = [arr[(P[i] + a) * Bf[f]:(P[i] + b) * Bf[f]] for (i, _, a, b) in h["chunks"]]
            per_field.append(np.concatenate(parts) if parts else np.zeros(0, dtype=np.uint8))
        out[r] = per_field
    return out


# ---------------------------------------------------------------------------
# step 6: routing
# ---------------------------------------------------------------------------

def route(src, dst, seq_lens, world):
    """Step 6: the decentralized plan.  One record per (i, overlap [x,y), dst replica td)
    (reading c19: uncoalesced), source replica ts = td mod TP_src (reading c9), canonical order
    (s, d, i, x).

    Record = (s, d, i, x, y, src_off, dst_off): token range [x,y) of sequence i goes from
    local token offset src_off on rank s to local token offset dst_off on rank d.
    """
    N = len(seq_lens)
    validate_layout(src, N, world)
    validate_layout(dst, N, world)
    validate_lengths(seq_lens)
    gs = assign_groups(src, seq_lens)
    gd = assign_groups(dst, seq_lens)
    hs = holdings(src, seq_lens, gs)
    hd = holdings(dst, seq_lens, gd)
    cs_of = seq_chunks(src, seq_lens, gs)
    cd_of = seq_chunks(dst, seq_lens, gd)
    segs = []
    for i in range(N):
        for (cd, a_d, b_d, kd) in cd_of[i]:
            for (cs, a_s, b_s, ks) in cs_of[i]:
                x, y = max(a_s, a_d), min(b_s, b_d)
                if x >= y:
                    continue
                for td in range(dst["tp"]):
                    ts = td % src["tp"]
                    s = rank_of(src, gs[i], ks, ts)
                    d = rank_of(dst, gd[i], kd, td)
                    src_off = hs[s]["local_off"][(i, cs)] + (x - a_s)
                    dst_off = hd[d]["local_off"][(i, cd)] + (x - a_d)
                    segs.append((s, d, i, x, y, src_off, dst_off))
    segs.sort(key=lambda r: (r[0], r[1], r[2], r[3]))
    return segs


def check_capacity(dst, seq_lens, g_of):
    """Reading c12: cu_seqlens is int32 and must not exceed INT32_MAX."""
    for r, h in holdings(dst, seq_lens, g_of).items():
        if h["n_tokens"] > INT32_MAX:
            raise OracleError(ERR_CAPACITY, f"rank {r} would hold {h['n_tokens']} tokens")


# ---------------------------------------------------------------------------
# steps 7-8: messages and assembly
# ---------------------------------------------------------------------------

def build_messages(segs, src_arrays, fields):
    """Step 7: for every (s, d) with s != d, the field-major concatenation of its segments' bytes
    (taken from rank s's own arrays: the data leaves from its computation origin)."""
    Bf = field_bytes(fields)
    msgs = {}
    keys = sorted({(r[0], r[1]) for r in segs if r[0] != r[1]})
    for (s, d) in keys:
        mine = [r for r in segs if r[0] == s and r[1] == d]
        parts = []
        for f in range(len(fields)):
            for (_, _, _, x, y, so, _) in mine:
                parts.append(src_arrays[s][f][so * Bf[f]:(so + y - x) * Bf[f]])
        msgs[(s, d)] = np.concatenate(parts) if parts else np.zeros(0, dtype=np.uint8)
    return msgs


def assemble(segs, msgs, src_arrays, dst, seq_lens, world, fields):
    """Step 8: every destination d writes each received segment at byte offset
    dst_off * B_f of field f (self segments are copied locally, at no link cost)."""
    Bf = field_bytes(fields)
    gd = assign_groups(dst, seq_lens)
    hd = holdings(dst, seq_lens, gd)
    out = {r: [np.zeros(h["n_tokens"] * Bf[f], dtype=np.uint8) for f in range(len(fields))]
           for r, h in hd.items()}
    written = {r: [np.zeros(h["n_tokens"], dtype=np.int64) for _ in fields] for r, h in hd.items()}
    cursor = {key: 0 for key in msgs}
    # message parsing: within a message, field-major, segments in canonical order
    for (s, d), m in msgs.items():
        mine = [r for r in segs if r[0] == s and r[1] == d]
        pos = 0
        for f in range(len(fields)):
            for (_, _, _, x, y, _, do) in mine:
                n = (y - x) * Bf[f]
                out[d][f][do * Bf[f]:do * Bf[f] + n] = m[pos:pos + n]
                written[d][f][do:do + y - x] += 1
                pos += n
        cursor[(s, d)] = pos
        assert pos == m.size
    for (s, d, _, x, y, so, do) in segs:
        if s == d:
            for f in range(len(fields)):
                n = (y - x) * Bf[f]
                out[d][f][do * Bf[f]:do * Bf[f] + n] = src_arrays[s][f][so * Bf[f]:so * Bf[f] + n]
                written[d][f][do:do + y - x] += 1
    # exactly-once at every destination replica (SURVEY.md §8(c) invariant)
    for r in written:
        for f in range(len(fields)):
            if written[r][f].size and not np.all(written[r][f] == 1):
                raise AssertionError(f"rank {r} field {f}: a token was written != 1 times")
    return out


def dispatch(src, dst, seq_lens, src_arrays, fields, world):
    """Steps 1-8: decentralized dispatch.  Returns (dst arrays per rank, meta per rank, plan)."""
    seq_lens = [int(x) for x in seq_lens]
    segs = route(src, dst, seq_lens, world)
    gd = assign_groups(dst, seq_lens)
    check_capacity(dst, seq_lens, gd)
    msgs = build_messages(segs, src_arrays, fields)
    out = assemble(segs, msgs, src_arrays, dst, seq_lens, world, fields)
    hd = holdings(dst, seq_lens, gd)
    meta = {r: {"cu_seqlens": h["cu_seqlens"], "seq_ids": h["seq_ids"], "tok_start": h["tok_start"]}
            for r, h in hd.items()}
    return out, meta, segs


# ---------------------------------------------------------------------------
# step 9: brute force (centralized gather-then-scatter)
# ---------------------------------------------------------------------------

def brute_force(src, dst, seq_lens, src_arrays, fields, world):
    """Step 9: rebuild the global per-field arrays from the src ranks (replica ts = 0, chunks in
    position order), then cut every dst rank's arrays straight out of them."""
    seq_lens = [int(x) for x in seq_lens]
    Bf = field_bytes(fields)
    gs = assign_groups(src, seq_lens)
    gd = assign_groups(dst, seq_lens)
    hs = holdings(src, seq_lens, gs)
    cs_of = seq_chunks(src, seq_lens, gs)
    glob = []
    for f in range(len(fields)):
        parts = []
        for i in range(len(seq_lens)):
            for (c, a, b, k) in cs_of[i]:
                r = rank_of(src, gs[i], k, 0)
                o = hs[r]["local_off"][(i, c)]
                parts.append(src_arrays[r][f][o * Bf[f]:(o + b - a) * Bf[f]])
        glob.append(np.concatenate(parts) if parts else np.zeros(0, dtype=np.uint8))
    return rank_arrays_from_global(dst, seq_lens, gd, glob, fields), glob


# ---------------------------------------------------------------------------
# step 10: stats, baseline
# ---------------------------------------------------------------------------

def stats(segs, fields, world):
    """Step 10: per-rank egress / ingress / self bytes, C[W][W] bytes,
    totals, segment count and coalesced-run count (runs with the same (s,d) whose src and dst
    token offsets are both contiguous, reading c19)."""
    B = sum(field_bytes(fields))
    C = [[0] * world for _ in range(world)]
    for (s, d, _, x, y, _, _) in segs:
        C[s][d] += (y - x) * B
    egress = [sum(C[s][d] for d in range(world) if d != s) for s in range(world)]
    ingress = [sum(C[s][d] for s in range(world) if s != d) for d in range(world)]
    self_b = [C[r][r] for r in range(world)]
    runs = 0
    prev = None
    for (s, d, _, x, y, so, do) in segs:
        if prev is not None and prev[0] == s and prev[1] == d and prev[2] == so and prev[3] == do:
            pass
        else:
            runs += 1
        prev = (s, d, so + (y - x), do + (y - x))
    return {
        "C": C,
        "egress": egress,
        "ingress": ingress,
        "self": self_b,
        "moved": sum(egress),
        "total": sum(sum(row) for row in C),
        "max_egress": max(egress) if egress else 0,
        "max_ingress": max(ingress) if ingress else 0,
        "segments": len(segs),
        "runs": runs,
    }


def gather_scatter_layouts(n_seqs, controller=0):
    """Centralized baseline (PAPER.md:163 'aggregated on a single node before redistribution';
    reading c13): every sequence first goes to DP1 on the controller rank,
    then from there to the destination layout.  Returns the middle layout."""
    return {"rank0": controller, "dp": 1, "sp": 1, "tp": 1, "assign": "given_counts",
            "counts": [int(n_seqs)], "group_of_seq": None}


def inverse_layouts(src, dst, seq_lens):
    """Round trip: the inverse dispatch uses dst as an EXPLICIT src layout and
    the original src as an EXPLICIT dst layout."""
    gs = assign_groups(src, seq_lens)
    gd = assign_groups(dst, seq_lens)
    inv_src = dict(dst, assign="explicit", counts=None, group_of_seq=np.asarray(gd, dtype=np.int32))
    inv_dst = dict(src, assign="explicit", counts=None, group_of_seq=np.asarray(gs, dtype=np.int32))
    return inv_src, inv_dst


def plan_hash(segs):
    """Determinism pin: a digest of the canonical plan."""
    h = hashlib.blake2b(digest_size=16)
    for r in segs:
        h.update(np.asarray(r, dtype=np.int64).tobytes())
    return h.hexdigest()


def lpt_exhaustive_opt(seq_lens, D):
    """Brute-force optimum makespan for tiny inputs (pin for LPT's Graham bound)."""
    best = None
    for assign in itertools.product(range(D), repeat=len(seq_lens)):
        loads = [0] * D
        for i, g in enumerate(assign):
            loads[g] += int(seq_lens[i])
        m = max(loads)
        best = m if best is None else min(best, m)
    return best


def group_loads(g_of, seq_lens, D):
    loads = [0] * D
    for i, g in enumerate(g_of):
        loads[g] += int(seq_lens[i])
    return loads


# ---------------------------------------------------------------------------
# NEXT-2: per-sequence fields (reading n4) and distributed advantage estimation (reading n5)
# ---------------------------------------------------------------------------

def seq_holdings(lay, seq_lens, g_of):
    """Every rank (g, k, t) of a layout holds one record per sequence of its group, ascending i
    -- every SP rank and TP replica holds a copy (reading n4).  rank -> [i, ...]."""
    out = {}
    for g, members in group_members(seq_lens, g_of, lay["dp"]).items():
        for k in range(lay["sp"]):
            for t in range(lay["tp"]):
                out[rank_of(lay, g, k, t)] = list(members)
    return out


def dispatch_seq_fields(src, dst, seq_lens, src_seq_arrays, sfields, world):
    """Route per-sequence fields (rewards, returns) with their sequences:
    destination rank d = (g, k, t) receives, at the position of sequence i in its group, the
    record the source holds for i -- read from source rank (g_src(i), SP 0, t mod TP_src), as for
    per-token fields (reading c9; all source copies are equal)."""
    seq_lens = [int(x) for x in seq_lens]
    validate_layout(src, len(seq_lens), world)
    validate_layout(dst, len(seq_lens), world)
    gs = assign_groups(src, seq_lens)
    gd = assign_groups(dst, seq_lens)
    hs = seq_holdings(src, seq_lens, gs)
    hd = seq_holdings(dst, seq_lens, gd)
    Bs = field_bytes(sfields)
    out = {}
    for d, members in hd.items():
        _, _, td = coords_of(dst, d)
        per_field = []
        for f in range(len(sfields)):
            parts = []
            for i in members:
                s = rank_of(src, gs[i], 0, td % src["tp"])
                p = hs[s].index(i)
                parts.append(src_seq_arrays[s][f][p * Bs[f]:(p + 1) * Bs[f]])
            per_field.append(np.concatenate(parts) if parts else np.zeros(0, dtype=np.uint8))
        out[d] = per_field
    return out


def discounted_returns(r, m, gamma):
    """Reading n5: G_t = m_t r_t + gamma G_{t+1} over one sequence, G_L = 0 (fp64).
    m is the boolean response mask: any nonzero byte is m_t = 1 (as in the statistics)."""
    G = np.zeros(len(r), dtype=np.float64)
    nxt = 0.0
    for t in range(len(r) - 1, -1, -1):
        nxt = (1.0 if m[t] else 0.0) * float(r[t]) + gamma * nxt
        G[t] = nxt
    return G


def distributed_advantages(src, seq_lens, rewards, masks, gamma, eps, world):
    """Reading n5 (REINFORCE++-style globally normalised returns), computed
    where the rollout holds the tokens (src layout, sp == 1) with no controller:
      1. every source rank: per sequence, G_t = m_t r_t + gamma G_{t+1};
      2. batch statistics over masked tokens (TP replica 0 counted once):
         mu = sum m G / sum m, sigma = sqrt(sum m G^2 / sum m - mu^2);
      3. A_t = m_t (G_t - mu) / (sigma + eps).
    rewards / masks: rank -> fp32 / u8 token arrays.  Returns (G, A, seq_return, stats)."""
    if src["sp"] != 1:
        raise OracleError(ERR_UNSUPPORTED, "returns need whole sequences on the source")
    seq_lens = [int(x) for x in seq_lens]
    gs = assign_groups(src, seq_lens)
    hs = holdings(src, seq_lens, gs)
    G, R = {}, {}
    n = s1 = s2 = 0.0
    for rank, h in hs.items():
        g_r = np.zeros(h["n_tokens"], dtype=np.float64)
        ret = []
        for (i, c, lo, hi) in h["chunks"]:
            o = h["local_off"][(i, c)]
            g_r[o:o + hi - lo] = discounted_returns(rewards[rank][o:o + hi - lo],
                                                    masks[rank][o:o + hi - lo], gamma)
            ret.append(g_r[o] if hi > lo else 0.0)
        G[rank], R[rank] = g_r, np.array(ret, dtype=np.float64)
        if coords_of(src, rank)[2] == 0:
            mk = masks[rank].astype(bool)
            n += float(mk.sum())
            s1 += float(g_r[mk].sum())
            s2 += float((g_r[mk] ** 2).sum())
    mu = s1 / n if n else 0.0
    var = max(s2 / n - mu * mu, 0.0) if n else 0.0
    sigma = var ** 0.5
    A = {rank: np.where(masks[rank].astype(bool), (G[rank] - mu) / (sigma + eps), 0.0)
         for rank in G}
    return G, A, R, (n, s1, s2)
