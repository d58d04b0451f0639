"""Pins for the SP split variants of the oracle (readings n1 zigzag, n2 flat,
n3 threshold): hand-worked golden holdings (tests/golden/sp_variants.json), an independently
written per-token owner model, and random layouts against the brute force / round trip."""
import json
import os
import random

import numpy as np
import pytest

from oracle import earl_oracle as O
from paper_2510_05943_b200 import workloads as W
from tests.helpers import random_layout

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "sp_variants.json")))


def lay(d):
    return W.layout(**d)


@pytest.mark.parametrize("case", sorted(GOLD["cases"]))
def test_golden_sp_variants(case):
    c = GOLD["cases"][case]
    lens = GOLD["lengths"]
    dst = lay(c["dst"])
    hd = O.holdings(dst, lens, O.assign_groups(dst, lens))
    for key in ("cu_seqlens", "tok_start"):
        for r, v in c[key].items():
            assert hd[int(r)][key] == v, (case, key, r)
    assert sum(h["n_tokens"] for h in hd.values()) == sum(lens)
    if "len16" in c:
        l16 = c["len16"]["lengths"]
        h16 = O.holdings(dst, l16, O.assign_groups(dst, l16))
        for r in (0, 1):
            assert [[lo, hi] for (_, _, lo, hi) in h16[r]["chunks"]] == c["len16"][f"chunks_rank{r}"]


# ---------------------------------------------------------------------------------------
# independent per-token owner model (written here, not with the oracle's helpers)
# ---------------------------------------------------------------------------------------

def block_sizes(n, parts):
    return [n // parts + (1 if j < n % parts else 0) for j in range(parts)]


def owner_of_token(layd, tok, L, pos_in_group, stream_pos, stream_total):
    SP = layd["sp"]
    split = layd.get("sp_split", "block")
    if split == "flat":
        edge = 0
        for k, sz in enumerate(block_sizes(stream_total, SP)):
            if edge <= stream_pos + tok < edge + sz:
                return k
            edge += sz
        raise AssertionError
    if split == "threshold" and L < layd.get("sp_min_len", 0):
        return pos_in_group % SP
    parts = 2 * SP if split == "zigzag" else SP
    edge = 0
    for j, sz in enumerate(block_sizes(L, parts)):
        if edge <= tok < edge + sz:
            return j if j < SP else 2 * SP - 1 - j
        edge += sz
    raise AssertionError


def per_token_holdings(layd, lens, groups, glob, Bfs):
    starts = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    out = {}
    for g in range(layd["dp"]):
        members = [i for i in range(len(lens)) if groups[i] == g]
        S = sum(int(lens[i]) for i in members)
        for k in range(layd["sp"]):
            toks = []
            spos = 0
            for p, i in enumerate(members):
                L = int(lens[i])
                for tok in range(L):
                    if owner_of_token(layd, tok, L, p, spos, S) == k:
                        toks.append(int(starts[i]) + tok)
                spos += L
            for t in range(layd["tp"]):
                r = layd["rank0"] + t + layd["tp"] * (k + layd["sp"] * g)
                out[r] = [np.array([glob[f][q * Bfs[f] + b] for q in toks for b in range(Bfs[f])],
                                   dtype=np.uint8) for f in range(len(Bfs))]
    return out


def with_split(rng, d):
    if d["sp"] > 1 or rng.random() < 0.3:
        split = rng.choice(["block", "zigzag", "flat", "threshold"])
        d = dict(d, sp_split=split, sp_min_len=rng.choice([0, 3, 10, 40]) if split == "threshold" else 0)
    return d


@pytest.mark.parametrize("seed", range(30))
def test_random_variant_layouts(seed):
    rng = random.Random(1000 + seed)
    world = rng.randint(1, 8)
    n = rng.randint(0, 18)
    lens = [rng.choice([0, 1, 2, 3, rng.randint(0, 60)]) for _ in range(n)]
    src = with_split(rng, random_layout(rng, world, n))
    dst = with_split(rng, random_layout(rng, world, n))
    fields = [("a", 4, 1, "x"), ("m", 1, 1, "x")]
    glob = W.gen_global_fields(fields, sum(lens), seed_base=seed, random_bits=True)
    src_arrays = O.rank_arrays_from_global(src, lens, O.assign_groups(src, lens), glob, fields)
    # the oracle's own holdings equal the per-token model on both sides
    pt_src = per_token_holdings(src, lens, O.assign_groups(src, lens), glob, O.field_bytes(fields))
    assert set(pt_src) == set(src_arrays)
    for r in pt_src:
        for f in range(len(fields)):
            assert np.array_equal(pt_src[r][f], src_arrays[r][f])
    out, meta, segs = O.dispatch(src, dst, lens, src_arrays, fields, world)
    bf, _ = O.brute_force(src, dst, lens, src_arrays, fields, world)
    pt = per_token_holdings(dst, lens, O.assign_groups(dst, lens), glob, O.field_bytes(fields))
    assert set(out) == set(bf) == set(pt)
    for r in out:
        for f in range(len(fields)):
            assert np.array_equal(out[r][f], bf[r][f])
            assert np.array_equal(out[r][f], pt[r][f])
        assert meta[r]["cu_seqlens"][-1] * O.field_bytes(fields)[0] == out[r][0].size
    inv_src, inv_dst = O.inverse_layouts(src, dst, lens)
    back, _, _ = O.dispatch(inv_src, inv_dst, lens, out, fields, world)
    for r in src_arrays:
        for f in range(len(fields)):
            assert np.array_equal(back[r][f], src_arrays[r][f])


def test_zigzag_balances_causal_attention_work():
    """Why zigzag (ring attention / context parallel): with causal attention the work of token t
    grows with t; zigzag gives every SP rank the same number of early and late tokens."""
    L, SP = 4096, 4
    d = W.layout(dp=1, sp=SP, assign="contig", sp_split="zigzag")
    h = O.holdings(d, [L], [0])
    work = [sum(sum(range(lo, hi)) for (_, _, lo, hi) in h[k]["chunks"]) for k in range(SP)]
    assert max(work) - min(work) <= L  # block would differ by ~L^2/SP
    b = O.holdings(W.layout(dp=1, sp=SP, assign="contig"), [L], [0])
    bwork = [sum(sum(range(lo, hi)) for (_, _, lo, hi) in b[k]["chunks"]) for k in range(SP)]
    assert max(bwork) - min(bwork) > 100 * L


def test_unknown_split_rejected():
    with pytest.raises(O.OracleError) as e:
        O.route(W.layout(dp=1), W.layout(dp=1, sp=2, sp_split="ring"), [4, 5], 2)
    assert e.value.code == O.ERR_INVALID_ARGUMENT
