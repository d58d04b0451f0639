"""Pins for NEXT-2 of the oracle: per-sequence fields routed with their sequences (reading n4)."""
import random

import numpy as np
import pytest

from oracle import earl_oracle as O
from paper_2510_05943_b200 import workloads as W
from tests.helpers import random_layout
from tests.test_oracle_sp_variants import with_split


def test_seq_fields_tiny_golden():
    """BASELINE configs[0] DP2 -> DP1 x SP2: both SP ranks list all 8 sequences, in order, so
    each receives the full per-sequence array (rank 0 held 0-3, rank 1 held 4-7)."""
    lens = W.TINY_LENGTHS.tolist()
    src = W.rollout_layout(8, 2)
    dst = W.layout(dp=1, sp=2, assign="contig")
    rewards = np.arange(8, dtype=np.float32) * 1.5
    sf = [("reward", 4, 1, "x")]
    src_arrays = {0: [rewards[:4].view(np.uint8)], 1: [rewards[4:].view(np.uint8)]}
    out = O.dispatch_seq_fields(src, dst, lens, src_arrays, sf, 2)
    for r in (0, 1):
        assert np.array_equal(out[r][0].view(np.float32), rewards)


@pytest.mark.parametrize("seed", range(25))
def test_seq_fields_equal_global_rows(seed):
    """Brute force: every destination rank's records are the global per-sequence rows of its
    group's sequences; distinct source replicas feed dst replica td from td mod TP_src."""
    rng = random.Random(seed)
    world = rng.randint(1, 8)
    n = rng.randint(0, 30)
    lens = [rng.randint(0, 50) for _ in range(n)]
    src = with_split(rng, random_layout(rng, world, n))
    dst = with_split(rng, random_layout(rng, world, n))
    sf = [("reward", 4, 1, "x"), ("meta", 1, 3, "x")]
    Bs = O.field_bytes(sf)
    # global rows, and a per-replica tag byte so each source replica differs
    glob = [np.random.default_rng(seed + f).integers(0, 256, size=n * Bs[f], dtype=np.uint8)
            for f in range(len(sf))]
    gs = O.assign_groups(src, lens)
    hs = O.seq_holdings(src, lens, gs)
    src_arrays = {}
    for r, members in hs.items():
        _, _, t = O.coords_of(src, r)
        arrs = []
        for f in range(len(sf)):
            rows = [glob[f][i * Bs[f]:(i + 1) * Bs[f]].copy() for i in members]
            for row in rows:
                row[0] ^= t  # replica t's copy carries its replica index in byte 0
            arrs.append(np.concatenate(rows) if rows else np.zeros(0, dtype=np.uint8))
        src_arrays[r] = arrs
    out = O.dispatch_seq_fields(src, dst, lens, src_arrays, sf, world)
    gd = O.assign_groups(dst, lens)
    for d, members in O.seq_holdings(dst, lens, gd).items():
        _, _, td = O.coords_of(dst, d)
        ts = td % src["tp"]
        for f in range(len(sf)):
            want = []
            for i in members:
                row = glob[f][i * Bs[f]:(i + 1) * Bs[f]].copy()
                row[0] ^= ts
                want.append(row)
            want = np.concatenate(want) if want else np.zeros(0, dtype=np.uint8)
            assert np.array_equal(out[d][f], want)


# ---------------------------------------------------------------------------------------
# reading n5: distributed returns / advantages
# ---------------------------------------------------------------------------------------

def test_discounted_returns_closed_forms():
    rng = np.random.default_rng(0)
    r = rng.standard_normal(50)
    m = (rng.random(50) < 0.8).astype(np.uint8)
    # gamma = 1: reversed cumulative sum of the masked rewards (a library routine)
    assert np.allclose(O.discounted_returns(r, m, 1.0), np.cumsum((r * m)[::-1])[::-1], atol=1e-12)
    # gamma = 0: the masked rewards themselves
    assert np.allclose(O.discounted_returns(r, m, 0.0), r * m, atol=0)
    # one terminal reward: a geometric sequence gamma^(L-1-t) R
    z = np.zeros(20)
    z[-1] = 3.0
    want = 3.0 * 0.9 ** (19 - np.arange(20))
    assert np.allclose(O.discounted_returns(z, np.ones(20), 0.9), want, rtol=1e-12)
    # the mask is boolean (reading n5): a byte of 2 or 255 selects the reward like 1 does
    m2 = m * np.where(rng.random(50) < 0.5, 2, 255).astype(np.uint8)
    assert np.array_equal(O.discounted_returns(r, m2, 0.9), O.discounted_returns(r, m, 0.9))


@pytest.mark.parametrize("seed", range(6))
def test_distributed_advantages_statistics(seed):
    rng = random.Random(seed)
    world = rng.randint(1, 8)
    n = rng.randint(1, 40)
    lens = [rng.randint(0, 80) for _ in range(n)]
    dp = rng.randint(1, world)
    tp = rng.randint(1, max(1, world // dp))
    src = W.layout(dp=dp, tp=tp, assign=rng.choice(["contig", "lpt"]))
    T = sum(lens)
    glob_r = np.random.default_rng(seed).standard_normal(T).astype(np.float32)
    glob_m = (np.random.default_rng(seed + 1).random(T) < 0.7).astype(np.uint8)
    fr = [("r", 4, 1, "x"), ("m", 1, 1, "x")]
    arrs = O.rank_arrays_from_global(src, lens, O.assign_groups(src, lens),
                                     [glob_r.view(np.uint8), glob_m], fr)
    rewards = {k: v[0].view(np.float32) for k, v in arrs.items()}
    masks = {k: v[1] for k, v in arrs.items()}
    G, A, R, (cnt, s1, s2) = O.distributed_advantages(src, lens, rewards, masks, 0.97, 1e-8, world)
    # the statistics equal numpy's mean / std over the batch's masked returns (replica 0 once)
    P = np.concatenate([[0], np.cumsum(lens)])
    allG = np.concatenate([O.discounted_returns(glob_r[P[i]:P[i + 1]], glob_m[P[i]:P[i + 1]], 0.97)
                           for i in range(n)]) if T else np.zeros(0)
    sel = glob_m.astype(bool)
    assert cnt == sel.sum()
    if cnt:
        assert np.isclose(s1 / cnt, allG[sel].mean(), rtol=1e-10, atol=1e-12)
        assert np.isclose(np.sqrt(max(s2 / cnt - (s1 / cnt) ** 2, 0)), allG[sel].std(), rtol=1e-8, atol=1e-10)
    # normalised advantages over the masked tokens: mean 0, std 1 (when the spread is real)
    a_all = np.concatenate([A[r][masks[r].astype(bool)] for r in A if O.coords_of(src, r)[2] == 0])
    if cnt > 3 and allG[sel].std() > 1e-3:
        assert abs(a_all.mean()) < 1e-9 and abs(a_all.std() - 1) < 1e-6
    # per-sequence return = G_0 of the sequence
    for rank, h in O.holdings(src, lens, O.assign_groups(src, lens)).items():
        for q, (i, c, lo, hi) in enumerate(h["chunks"]):
            if hi > lo:
                assert R[rank][q] == G[rank][h["local_off"][(i, c)]]
