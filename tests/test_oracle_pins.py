"""Pins for the CPU oracle (oracle/earl_oracle.py) against things other than itself.

* tests/golden/c1_tiny.json: hand-worked tiny case (BASELINE.json configs[0]).
* SPEC.md worked examples (SPEC.md:218-220 block_layout, 227-229 plan_all_to_all,
  237 plan_gather_scatter, 459 the 2*W modeled ratio).
* closed forms / textbook routines: exclusive scan == shifted cumsum; LPT vs exhaustive
  search within Graham's (4/3 - 1/(3D)) bound; CONTIG balance bound T/D + max L.
* an independently written per-token brute force (this file) for holdings + routing + assembly.
* invariants: exactly once, conservation, round trip, dominance, determinism.
"""
import json
import os
import random

import numpy as np
import pytest

from oracle import earl_oracle as O
from paper_2510_05943_b200 import workloads as W

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "c1_tiny.json")))


def lay(d):
    return W.layout(**{k: v for k, v in d.items()})


def tiny_fields():
    return [("f0", 4, 1, "ids"), ("f1", 4, 1, "x"), ("f2", 4, 1, "x")]


# ---------------------------------------------------------------------------
# independent per-token model (written here without the oracle's helpers)
# ---------------------------------------------------------------------------

def chunk_of_token(L, SP, tok):
    sizes = [L // SP + (1 if j < L % SP else 0) for j in range(SP)]
    edge = 0
    for j, s in enumerate(sizes):
        if edge <= tok < edge + s:
            return j, tok - edge
        edge += s
    raise AssertionError


def per_token_holdings(layd, lens, groups, glob, Bfs):
    """rank -> per-field bytes, by walking every token of every member sequence."""
    starts = [0]
    for x in lens:
        starts.append(starts[-1] + int(x))
    out = {}
    for g in range(layd["dp"]):
        for k in range(layd["sp"]):
            toks = []
            for i in range(len(lens)):
                if groups[i] != g:
                    continue
                for tok in range(int(lens[i])):
                    if chunk_of_token(int(lens[i]), layd["sp"], tok)[0] == k:
                        toks.append(starts[i] + tok)
            for t in range(layd["tp"]):
                r = layd["rank0"] + t + layd["tp"] * (k + layd["sp"] * g)
                out[r] = [np.array([glob[f][q * Bfs[f] + b] for q in toks for b in range(Bfs[f])],
                                   dtype=np.uint8) for f in range(len(Bfs))]
    return out


# ---------------------------------------------------------------------------
# golden tiny case
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("case", sorted(GOLD["cases"].keys()))
def test_golden_c1(case):
    c = GOLD["cases"][case]
    lens = GOLD["lengths"]
    src = lay(GOLD["src"])
    dst = lay(c["dst"])
    world = c["world"]
    fields = tiny_fields()
    assert O.field_bytes(fields) == GOLD["fields_bytes_per_token"]
    gd = O.assign_groups(dst, lens)
    if "groups" in c:
        assert gd == c["groups"]
    if "loads" in c:
        assert O.group_loads(gd, lens, dst["dp"]) == c["loads"]
    if "exhaustive_opt" in c:
        assert O.lpt_exhaustive_opt(lens, dst["dp"]) == c["exhaustive_opt"]
    hs = O.holdings(src, lens, O.assign_groups(src, lens))
    assert [hs[r]["n_tokens"] for r in range(2)] == GOLD["src_tokens_per_rank"]
    hd = O.holdings(dst, lens, gd)
    for key in ("cu_seqlens", "seq_ids", "tok_start"):
        for r, v in c.get(key, {}).items():
            assert hd[int(r)][key] == v, (key, r)
    segs = O.route(src, dst, lens, world)
    st = O.stats(segs, fields, world)
    if "C_tokens" in c:
        B = 12
        for s in range(len(c["C_tokens"])):
            for d in range(len(c["C_tokens"][s])):
                assert st["C"][s][d] == c["C_tokens"][s][d] * B, (s, d)
    if "moved_bytes" in c:
        assert st["moved"] == c["moved_bytes"]
    if "self_bytes" in c:
        assert sum(st["self"]) == c["self_bytes"]
    if "total_bytes" in c:
        assert st["total"] == c["total_bytes"]
    if "runs" in c:  # hand-counted coalesced runs (reading c19)
        assert st["runs"] == c["runs"], (case, st["runs"])


def test_block_split_spot_values():
    for L, SP, want in GOLD["block_split"]["cases"]:
        assert [list(O.sp_chunk(L, SP, k)) for k in range(SP)] == want


def test_block_split_partition_property():
    for L in range(0, 40):
        for SP in range(1, 9):
            ch = [O.sp_chunk(L, SP, k) for k in range(SP)]
            assert ch[0][0] == 0 and ch[-1][1] == L
            for k in range(SP - 1):
                assert ch[k][1] == ch[k + 1][0]
            sizes = [b - a for a, b in ch]
            assert max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True)


# ---------------------------------------------------------------------------
# SPEC.md worked examples (rows == sequences of length 1)
# ---------------------------------------------------------------------------

def test_spec_block_layout_examples():
    assert O.count_blocks(16, 4) == [4, 4, 4, 4]
    assert O.count_blocks(5, 2) == [3, 2]
    assert O.count_blocks(7, 1) == [7]


def test_spec_plan_all_to_all_2x8_to_4x4():
    lens = [1] * 16
    src = W.layout(dp=2, assign="given_counts", counts=[8, 8])
    dst = W.layout(dp=4, assign="given_counts", counts=[4, 4, 4, 4])
    segs = O.route(src, dst, lens, 4)
    moved = sorted((s, d, i) for (s, d, i, *_rest) in segs if s != d)
    want = sorted([(0, 1, i) for i in range(4, 8)] + [(1, 2, i) for i in range(8, 12)]
                  + [(1, 3, i) for i in range(12, 16)])
    assert moved == want
    assert len(moved) == 12


def test_spec_identity_is_empty_and_disjoint_moves_everything():
    lens = [3, 1, 4, 1, 5, 9, 2, 6]
    src = W.layout(dp=2, assign="given_counts", counts=[4, 4])
    segs = O.route(src, dict(src), lens, 2)
    assert O.stats(segs, tiny_fields(), 2)["moved"] == 0
    dst = W.layout(rank0=2, dp=2, assign="given_counts", counts=[4, 4])
    st = O.stats(O.route(src, dst, lens, 4), tiny_fields(), 4)
    assert st["moved"] == sum(lens) * 12


def test_spec_gather_scatter_32_rows():
    lens = [1] * 16
    src = W.layout(rank0=1, dp=2, assign="given_counts", counts=[8, 8])
    dst = W.layout(rank0=3, dp=2, assign="given_counts", counts=[8, 8])
    mid = O.gather_scatter_layouts(16, controller=0)
    f = [("row", 1, 1, "x")]
    p1 = O.stats(O.route(src, mid, lens, 5), f, 5)
    p2 = O.stats(O.route(mid, dst, lens, 5), f, 5)
    assert p1["moved"] == 16 and p2["moved"] == 16 and p1["moved"] + p2["moved"] == 32
    assert p1["ingress"][0] == 16 and p2["egress"][0] == 16


@pytest.mark.parametrize("world", [2, 4, 8])
def test_modeled_ratio_is_2W(world):
    """SPEC.md:459 acceptance #5 restated for NVLink (SURVEY.md §8(c) analytic pin): with equal
    payloads and nothing resident on the controller, t_gs / t_a2a = 2W."""
    per = world * 3
    lens = [7] * (per * world)
    src = W.layout(dp=world, assign="given_counts", counts=[per] * world)
    dst = W.layout(dp=world, assign="explicit",
                   group_of_seq=np.arange(per * world, dtype=np.int32) % world)
    f = [("x", 4, 1, "x")]
    a2a = O.stats(O.route(src, dst, lens, world), f, world)
    t_a2a = max(max(a2a["egress"]), max(a2a["ingress"]))
    # controller = rank 0: it serializes (W-1)*P in, then (W-1)*P out on its own link
    mid = O.gather_scatter_layouts(len(lens), controller=0)
    g1 = O.stats(O.route(src, mid, lens, world), f, world)
    g2 = O.stats(O.route(mid, dst, lens, world), f, world)
    t_gs = g1["ingress"][0] + g2["egress"][0]
    # uniform all-to-all: each rank keeps 1/W of its payload P and sends (W-1)/W of it
    P = per * 7 * 4
    assert t_a2a * world == P * (world - 1)
    assert t_gs == 2 * (world - 1) * P
    assert t_gs == 2 * world * t_a2a


# ---------------------------------------------------------------------------
# textbook routines and closed forms
# ---------------------------------------------------------------------------

def test_exclusive_scan_is_shifted_cumsum():
    rng = np.random.default_rng(5)
    for n in (0, 1, 7, 1000):
        L = rng.integers(0, 40000, size=n)
        P, T = O.exclusive_scan(L)
        cs = np.cumsum(L)
        assert P == ([0] + cs[:-1].tolist() if n else [])
        assert T == (int(cs[-1]) if n else 0)


def test_lpt_graham_bound_vs_exhaustive():
    rng = random.Random(11)
    for _ in range(60):
        n = rng.randint(1, 8)
        D = rng.randint(1, 3)
        L = [rng.randint(0, 50) for _ in range(n)]
        g = O.assign_lpt(L, D)
        mk = max(O.group_loads(g, L, D))
        opt = O.lpt_exhaustive_opt(L, D)
        assert opt <= mk <= (4 / 3 - 1 / (3 * D)) * opt + 1e-9


def test_lpt_greedy_invariant():
    """Each placement goes to a least-loaded group at that moment (the definition of LPT)."""
    rng = random.Random(2)
    L = [rng.randint(0, 9000) for _ in range(300)]
    D = 5
    g = O.assign_lpt(L, D)
    order = sorted(range(len(L)), key=lambda i: (-L[i], i))
    loads = [0] * D
    for i in order:
        assert loads[g[i]] == min(loads)
        assert g[i] == loads.index(min(loads))
        loads[g[i]] += L[i]


def test_contig_balance_and_order():
    rng = np.random.default_rng(3)
    for _ in range(50):
        n = int(rng.integers(1, 200))
        D = int(rng.integers(1, 9))
        L = rng.integers(0, 5000, size=n).tolist()
        g = O.assign_contig(L, D)
        assert all(g[i] <= g[i + 1] for i in range(n - 1))  # contiguous blocks, order kept
        assert all(0 <= x < D for x in g)
        T = sum(L)
        if T:
            for load in O.group_loads(g, L, D):
                assert load <= T / D + max(L)


# ---------------------------------------------------------------------------
# random layouts: decentralized == brute force == independent per-token model
# ---------------------------------------------------------------------------

def random_layout(rng, world, n):
    while True:
        dp = rng.randint(1, world)
        sp = rng.randint(1, max(1, world // dp))
        tp = rng.randint(1, max(1, world // (dp * sp)))
        if dp * sp * tp <= world:
            break
    rank0 = rng.randint(0, world - dp * sp * tp)
    a = rng.choice(["given_counts", "contig", "lpt", "explicit"])
    counts = gos = None
    if a == "given_counts":
        cuts = sorted(rng.randint(0, n) for _ in range(dp - 1))
        counts = [b - a_ for a_, b in zip([0] + cuts, cuts + [n])]
    if a == "explicit":
        gos = [rng.randrange(dp) for _ in range(n)]
    return W.layout(rank0=rank0, dp=dp, sp=sp, tp=tp, assign=a, counts=counts, group_of_seq=gos)


def make_src_arrays(src, lens, glob, fields):
    gs = O.assign_groups(src, lens)
    return O.rank_arrays_from_global(src, lens, gs, glob, fields)


@pytest.mark.parametrize("seed", range(40))
def test_random_layouts_dispatch_equals_brute_force(seed):
    rng = random.Random(seed)
    world = rng.randint(1, 8)
    n = rng.randint(0, 24)
    lens = [rng.choice([0, 1, 2, 3, rng.randint(0, 70)]) for _ in range(n)]
    src = random_layout(rng, world, n)
    dst = random_layout(rng, world, n)
    fields = [("a", 4, 1, "x"), ("b", 1, 1, "x"), ("c", 2, 3, "x")]
    T = sum(lens)
    glob = W.gen_global_fields(fields, T, seed_base=seed * 10, random_bits=True)
    src_arrays = make_src_arrays(src, lens, glob, fields)
    out, meta, segs = O.dispatch(src, dst, lens, src_arrays, fields, world)
    bf, glob2 = O.brute_force(src, dst, lens, src_arrays, fields, world)
    for f in range(len(fields)):
        assert np.array_equal(glob2[f], glob[f])
    assert set(out) == set(bf)
    for r in out:
        for f in range(len(fields)):
            assert np.array_equal(out[r][f], bf[r][f])
    # independent per-token model (holdings, chunking and rank order written separately)
    pt = per_token_holdings(dst, lens, O.assign_groups(dst, lens), glob, O.field_bytes(fields))
    assert set(pt) == set(out)
    for r in out:
        for f in range(len(fields)):
            assert np.array_equal(out[r][f], pt[r][f])
    # conservation: total = T * B * TP_dst; sum egress == sum ingress
    st = O.stats(segs, fields, world)
    assert st["total"] == T * sum(O.field_bytes(fields)) * dst["tp"]
    assert sum(st["egress"]) == sum(st["ingress"])
    # coverage of the plan: every (i, token, td) exactly once
    cover = {}
    for (s, d, i, x, y, so, do) in segs:
        for tok in range(x, y):
            key = (i, tok, O.coords_of(dst, d)[2])
            cover[key] = cover.get(key, 0) + 1
    assert len(cover) == T * dst["tp"] and set(cover.values()) <= {1}
    # dominance: a2a moves no more than gather-and-scatter
    mid = O.gather_scatter_layouts(n, controller=0)
    g1 = O.stats(O.route(src, mid, lens, world), fields, world)
    g2 = O.stats(O.route(mid, dst, lens, world), fields, world)
    assert st["moved"] <= g1["moved"] + g2["moved"]


@pytest.mark.parametrize("seed", range(15))
def test_round_trip_identity(seed):
    rng = random.Random(100 + seed)
    world = rng.randint(1, 8)
    n = rng.randint(0, 20)
    lens = [rng.randint(0, 40) for _ in range(n)]
    src = random_layout(rng, world, n)
    dst = random_layout(rng, world, n)
    fields = [("a", 4, 1, "x"), ("m", 1, 1, "x")]
    glob = W.gen_global_fields(fields, sum(lens), seed_base=seed, random_bits=True)
    src_arrays = make_src_arrays(src, lens, glob, fields)
    out, _, _ = O.dispatch(src, dst, lens, src_arrays, fields, world)
    inv_src, inv_dst = O.inverse_layouts(src, dst, lens)
    back, _, _ = O.dispatch(inv_src, inv_dst, lens, out, fields, world)
    assert set(back) == set(src_arrays)
    for r in back:
        for f in range(len(fields)):
            assert np.array_equal(back[r][f], src_arrays[r][f])


def test_determinism_plan_hash():
    lens = W.c2_lengths(0)[:64].tolist()
    src = W.rollout_layout(64, 8)
    dst = W.layout(dp=2, tp=4, assign="contig")
    h1 = O.plan_hash(O.route(src, dst, lens, 8))
    h2 = O.plan_hash(O.route(src, dst, list(lens), 8))
    assert h1 == h2
    lens[3] += 1
    assert O.plan_hash(O.route(src, dst, lens, 8)) != h1


def test_zero_lengths_and_empty_ranks():
    lens = [0, 0, 5, 0]
    src = W.layout(dp=2, assign="given_counts", counts=[2, 2])
    dst = W.layout(dp=4, sp=2, assign="given_counts", counts=[0, 1, 3, 0])
    out, meta, segs = O.dispatch(src, dst, lens, make_src_arrays(src, lens, W.gen_global_fields(
        tiny_fields(), 5, random_bits=True), tiny_fields()), tiny_fields(), 8)
    assert meta[0]["cu_seqlens"] == [0] and meta[0]["seq_ids"] == []
    assert meta[2]["cu_seqlens"] == [0, 0] and meta[3]["cu_seqlens"] == [0, 0]
    assert meta[4]["cu_seqlens"] == [0, 0, 3, 3] and meta[5]["cu_seqlens"] == [0, 0, 2, 2]
    assert meta[5]["tok_start"] == [0, 3, 0]
    assert len(segs) == 2


# ---------------------------------------------------------------------------
# errors (§8(b) status list)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("bad,code", [
    (dict(dp=3, tp=3), O.ERR_LAYOUT),                                   # 9 ranks > W
    (dict(dp=2, assign="given_counts", counts=[1, 1]), O.ERR_LAYOUT),    # sum != N
    (dict(dp=2, assign="explicit", group_of_seq=[0, 2, 0, 0]), O.ERR_LAYOUT),
    (dict(rank0=7, dp=2), O.ERR_LAYOUT),
])
def test_layout_errors(bad, code):
    with pytest.raises(O.OracleError) as e:
        O.route(W.layout(dp=1), W.layout(**bad), [1, 2, 3, 4], 8)
    assert e.value.code == code


def test_other_errors():
    with pytest.raises(O.OracleError) as e:
        O.route(W.layout(dp=1), W.layout(dp=1), [1, -2], 8)
    assert e.value.code == O.ERR_INVALID_ARGUMENT
    with pytest.raises(O.OracleError) as e:
        O.route(W.layout(dp=1), W.layout(dp=2, assign="lpt"), [1] * 8193, 8)
    assert e.value.code == O.ERR_CAPACITY
    with pytest.raises(O.OracleError) as e:
        O.route(W.layout(dp=1), W.layout(dp=1), [1], 9)
    assert e.value.code == O.ERR_UNSUPPORTED


def test_capacity_boundary_int32_cu_seqlens():
    """Reading c12: cu_seqlens is int32, so a destination shard may hold at most INT32_MAX =
    2^31 - 1 tokens (a number fixed by the int32 type, not by the oracle).  Exactly at the
    boundary passes; one token more raises CAPACITY.  Lengths only: holdings are counts."""
    edge = 2**31 - 1
    dp1 = W.layout(dp=1, assign="contig")
    O.check_capacity(dp1, [2**30, 2**30 - 1], [0, 0])          # 2^31 - 1 tokens: fits
    with pytest.raises(O.OracleError) as e:
        O.check_capacity(dp1, [2**30, 2**30], [0, 0])          # 2^31: one too many
    assert e.value.code == O.ERR_CAPACITY
    with pytest.raises(O.OracleError) as e:
        O.check_capacity(dp1, [2**20] * 2049, [0] * 2049)      # 2049 x 2^20 = 2^31 + 2^20
    assert e.value.code == O.ERR_CAPACITY
    # SP2 splits every sequence, the earlier chunk taking the odd token (reading c7):
    # SP rank 0 holds 2^30 of 2^31 - 1 plus 2^30 - 1 of 2^31 - 3 = 2^31 - 1 tokens
    sp2 = W.layout(dp=1, sp=2, assign="contig")
    O.check_capacity(sp2, [edge, edge - 2], [0, 0])
    with pytest.raises(O.OracleError):
        O.check_capacity(sp2, [edge, edge], [0, 0])           # SP rank 0: 2^30 + 2^30
    # DP2: the same 2^31 tokens split over two groups fit
    dp2 = W.layout(dp=2, assign="contig")
    lens = [2**30, 2**30]
    O.check_capacity(dp2, lens, O.assign_groups(dp2, lens))
    # TP replicas each hold the whole group: replication does not change the per-rank count
    tp4 = W.layout(dp=1, tp=4, assign="contig")
    O.check_capacity(tp4, [edge], [0])
    with pytest.raises(O.OracleError):
        O.check_capacity(tp4, [edge, 1], [0, 0])


@pytest.mark.parametrize("seed", range(12))
def test_contig_without_sp_is_one_run_per_pair(seed):
    """Reading c19 + SPEC.md:262: under monotone layouts without SP (rollout GIVEN_COUNTS ->
    CONTIG, TP replicas allowed) every (s, d) pair's segments are one contiguous run on both sides,
    so the coalesced run count equals the number of (s, d) pairs with bytes, and it never exceeds
    SPEC's coalescing bound |src ranges| + |dst ranges| per replica pair."""
    rng = random.Random(seed)
    world = rng.randint(1, 8)
    n = rng.randint(1, 40)
    lens = [rng.randint(0, 50) for _ in range(n)]
    sdp = rng.randint(1, world)
    stp = rng.randint(1, world // sdp)
    ddp = rng.randint(1, world)
    dtp = rng.randint(1, world // ddp)
    src = W.layout(dp=sdp, tp=stp, assign="given_counts", counts=O.count_blocks(n, sdp))
    dst = W.layout(dp=ddp, tp=dtp, assign="contig")
    segs = O.route(src, dst, lens, world)
    st = O.stats(segs, [("a", 4, 1, "x")], world)
    pairs = {(s, d) for (s, d, _, x, y, _, _) in segs}
    assert st["runs"] == len(pairs)
    assert st["runs"] <= (sdp + ddp) * dtp


def test_golden_tp_replica_rule():
    lens = GOLD["lengths"]
    for c in GOLD["tp_replica_cases"]["cases"]:
        st = O.stats(O.route(lay(c["src"]), lay(c["dst"]), lens, c["world"]), tiny_fields(), c["world"])
        for s, row in enumerate(c["C_tokens"]):
            for d, v in enumerate(row):
                assert st["C"][s][d] == v * 12, (s, d)


def test_distinct_src_replicas_feed_td_mod_tps():
    """Give every src replica distinct bytes; dst replica td must equal src replica td % TP_src."""
    lens = [3, 0, 7, 2, 9]
    fields = [("a", 4, 1, "x"), ("m", 1, 1, "x")]
    for tps, tpd in [(2, 4), (4, 2), (3, 2), (2, 3)]:
        src = W.layout(dp=1, tp=tps, assign="contig")
        dst = W.layout(dp=1, sp=1, tp=tpd, assign="contig")
        src_arrays = {t: [W.gen_field_bytes(f, sum(lens), 50 + 7 * t + k, True) for k, f in enumerate(fields)]
                      for t in range(tps)}
        out, _, _ = O.dispatch(src, dst, lens, src_arrays, fields, 8)
        for td in range(tpd):
            for f in range(len(fields)):
                assert np.array_equal(out[td][f], src_arrays[td % tps][f])


def test_fig4_workload_matches_the_papers_payloads():
    """tests/golden/paper_numbers.json: the Fig. 4 replay's per-worker log-prob
    payload is the paper's 46 / 93 / 187 MiB (printed rounded down) at 8K / 16K / 32K."""
    import json
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_numbers.json")))["fig4"]
    for L, mib in zip(g["contexts"], g["per_worker_MiB"]):
        lens = W.fig4_lengths(L, 8)
        counts = W.near_equal_counts(len(lens), 8)
        per_worker = W.rollout_token_counts(lens, counts)
        assert len(set(per_worker)) == 1
        assert int(per_worker[0] * 4 / (1 << 20)) == mib


def test_table1_is_linear_in_context():
    """Table 1: the estimated batch grows linearly with the context length,
    15,625 MiB per 1K tokens on a 1K-GPU cluster (kappa of SPEC.md:59)."""
    import json
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_numbers.json")))["table1"]
    for L, mib in zip(g["contexts"], g["MiB"]):
        assert mib * 1024 == 15625 * L
