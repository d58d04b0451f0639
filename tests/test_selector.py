"""NEXT-4 host side: the Parallelism Selector (Eq. (1)).

The oracle (oracle/selector_oracle.py) is pinned to the paper's numbers, SPEC.md's worked
examples and invariants; then the library's C ABI (earl_speedup_pct / earl_policy_*; host code,
no GPU) must agree with it on random profiles.  All CPU."""
import itertools
import random

import numpy as np
import pytest

from oracle import selector_oracle as S

K = 1024
BOUNDS = [0, 8 * K, 16 * K, 32 * K, 64 * K]  # reading s1: powers-of-two context ranges
TP = [4, 8]
# Fig. 3, 32 responses: TP4 31% faster at short context, TP8 5% faster at
# 16K and 32K; 128 responses: TP4 OOM at 32K
FIG3 = [[131.0, 100.0, 100.0, 100.0],   # TP4
        [100.0, 105.0, 105.0, 105.0]]   # TP8


# ---- oracle pins ---------------------------------------------------------------------------

def test_speedup_examples():
    assert S.speedup_pct(100, 100) == 0.0
    assert S.speedup_pct(100, 131) == pytest.approx(31.0)   # "31% higher throughput"
    assert S.speedup_pct(200, 210) == pytest.approx(5.0)    # "yields 5% improvement"
    with pytest.raises(S.SelectorError):
        S.speedup_pct(0, 1)


def test_speedup_antisymmetry():
    rng = random.Random(0)
    for _ in range(200):
        a, b = rng.uniform(1, 1e4), rng.uniform(1, 1e4)
        s = S.speedup_pct(a, b)
        assert S.speedup_pct(b, a) == pytest.approx(-100 * s / (100 + s), rel=1e-9, abs=1e-9)


def test_fig3_policy_switches_to_tp8_at_16k():
    assert S.build_policy(TP, BOUNDS, FIG3) == [0, 1, 1, 1]
    assert S.select([0, 1, 1, 1], BOUNDS, 0, 4000, 0) == (0, False)
    assert S.select([0, 1, 1, 1], BOUNDS, 0, 17000, 0) == (1, True)   # "switches to TP=8"


def test_oom_entries_are_never_selected():
    tgs = [[131.0, 100.0, 120.0, 200.0], [100.0, 105.0, 105.0, 105.0]]
    oom = [[0, 0, 0, 1], [0, 0, 0, 0]]   # TP4 OOMs at 32K with 128 responses
    assert S.build_policy(TP, BOUNDS, tgs, oom) == [0, 1, 0, 1]
    with pytest.raises(S.SelectorError) as e:
        S.build_policy(TP, BOUNDS, tgs, [[0, 0, 0, 1], [0, 0, 0, 1]])
    assert e.value.kind == "policy"


def test_tie_goes_to_smaller_tp_in_any_order():
    tgs = {4: [100.0, 50.0], 8: [100.0, 60.0], 2: [90.0, 60.0]}
    for perm in itertools.permutations([4, 8, 2]):
        table = S.build_policy(list(perm), [0, 10, 20], [tgs[t] for t in perm])
        assert [perm[c] for c in table] == [4, 2]


def test_argmax_invariant_under_scaling():
    rng = random.Random(1)
    for _ in range(50):
        nc, nb = rng.randint(1, 5), rng.randint(1, 6)
        tgs = [[rng.choice([1.0, 2.0, 3.0, rng.uniform(1, 9)]) for _ in range(nb)] for _ in range(nc)]
        tp = [rng.choice([1, 2, 4, 8]) for _ in range(nc)]
        bounds = list(range(0, 100 * (nb + 1), 100))
        k = rng.choice([0.5, 3.0, 1e3])
        assert S.build_policy(tp, bounds, tgs) == S.build_policy(tp, bounds, [[x * k for x in r] for r in tgs])


def test_hysteresis_holds_the_current_config_near_a_boundary():
    table = S.build_policy(TP, BOUNDS, FIG3)
    cur, switches = 0, 0
    for x in [8150, 8250] * 5:           # oscillation across the 8K boundary
        cur, sw = S.select(table, BOUNDS, 500, x, cur)
        switches += sw
    assert cur == 0 and switches == 0
    # without hysteresis the same trace switches on every step
    cur, switches = 0, 0
    for x in [8150, 8250] * 5:
        cur, sw = S.select(table, BOUNDS, 0, x, cur)
        switches += sw
    assert switches == 9   # every observation after the first crosses the boundary
    # beyond the band it switches once and stays
    assert S.select(table, BOUNDS, 500, 9000, 0) == (1, True)
    assert S.select(table, BOUNDS, 500, 8000, 1) == (1, False)   # 192 tokens below the edge
    assert S.select(table, BOUNDS, 500, 7000, 1) == (0, True)


def test_hysteresis_never_keeps_an_oom_configuration():
    """Reading s2 + s3: hysteresis keeps the current configuration near a boundary, but never
    into a range where it runs out of memory (TP4 OOM at long context).  Fig. 3
    with TP4 OOM from 8K on: at 8.2K (200 tokens past the edge, hysteresis 500) the plain
    hysteresis rule keeps TP4; with the OOM mask it must switch to TP8."""
    tgs = [[131.0, 100.0, 100.0, 100.0], [100.0, 105.0, 105.0, 105.0]]
    bounds = [0, 8 * K, 16 * K, 32 * K, 64 * K]
    oom_from_8k = [[0, 1, 1, 1], [0, 0, 0, 0]]
    oom_from_16k = [[0, 0, 1, 1], [0, 0, 0, 0]]
    table = S.build_policy(TP, bounds, tgs, oom_from_8k)
    assert table == [0, 1, 1, 1] == S.build_policy(TP, bounds, tgs, oom_from_16k)
    assert S.select(table, bounds, 500, 8 * K + 200, 0) == (0, False)               # plain s3
    assert S.select(table, bounds, 500, 8 * K + 200, 0, oom_from_16k) == (0, False)  # TP4 fits
    assert S.select(table, bounds, 500, 8 * K + 200, 0, oom_from_8k) == (1, True)    # TP4 OOMs
    earl = _lib()
    p = earl.Policy(TP, bounds, tgs, oom_from_8k, 500)
    assert p.select(8 * K + 200, 0) == (1, True)
    p.destroy()


def test_hysteresis_bound_at_most_one_switch_within_a_band():
    rng = random.Random(2)
    table = S.build_policy(TP, BOUNDS, FIG3)
    for _ in range(100):
        cur = rng.randrange(2)
        switches = 0
        for _ in range(30):
            cur, sw = S.select(table, BOUNDS, 400, rng.uniform(8 * K - 399, 8 * K + 399), cur)
            switches += sw
        assert switches <= 1


def test_observe_is_the_mean():
    assert S.observe([4000, 6000]) == 5000
    assert S.observe([777] * 9) == 777
    with pytest.raises(S.SelectorError):
        S.observe([])
    with pytest.raises(S.SelectorError):
        S.bucket_of(BOUNDS, 64 * K)


# ---- the library (C ABI, host code) against the oracle ---------------------------------------

def _lib():
    from paper_2510_05943_b200 import build
    build.build()
    from paper_2510_05943_b200 import earl
    return earl


def test_library_speedup_and_errors():
    earl = _lib()
    assert earl.speedup_pct(100, 131) == pytest.approx(31.0)
    with pytest.raises(earl.EarlError) as e:
        earl.speedup_pct(-1, 2)
    assert e.value.name == "EARL_ERR_INVALID_ARGUMENT"
    with pytest.raises(earl.EarlError) as e:
        earl.Policy(TP, BOUNDS, FIG3, [[1] * 4, [0, 0, 1, 0]])
    assert e.value.name == "EARL_ERR_POLICY" and "range 2" in str(e.value)
    p = earl.Policy(TP, BOUNDS, FIG3)
    with pytest.raises(earl.EarlError) as e:
        p.select(64 * K, 0)
    assert e.value.name == "EARL_ERR_POLICY"
    with pytest.raises(earl.EarlError) as e:
        p.select(100, 2)
    assert e.value.name == "EARL_ERR_INVALID_ARGUMENT"
    with pytest.raises(earl.EarlError):
        earl.Policy(TP, [0, 10, 10], [[1, 1], [1, 1]])


@pytest.mark.parametrize("seed", range(40))
def test_library_policy_matches_oracle(seed):
    earl = _lib()
    rng = random.Random(100 + seed)
    nc, nb = rng.randint(1, 6), rng.randint(1, 8)
    tp = [rng.choice([1, 2, 4, 8]) for _ in range(nc)]
    edges = sorted(rng.sample(range(1, 200_000), nb))
    bounds = [0] + edges
    nb = len(bounds) - 1
    tgs = [[float(rng.choice([10, 20, 30, rng.randint(1, 40)])) for _ in range(nb)] for _ in range(nc)]
    oom = [[int(rng.random() < 0.25) for _ in range(nb)] for _ in range(nc)]
    hyst = rng.choice([0, 100, 1000, 5000])
    try:
        want = S.build_policy(tp, bounds, tgs, oom)
    except S.SelectorError:
        with pytest.raises(earl.EarlError) as e:
            earl.Policy(tp, bounds, tgs, oom, hyst)
        assert e.value.name == "EARL_ERR_POLICY"
        return
    p = earl.Policy(tp, bounds, tgs, oom, hyst)
    assert p.table() == want
    cur = rng.randrange(nc)
    for _ in range(60):
        x = rng.uniform(bounds[0], bounds[-1] - 1e-6)
        got = p.select(x, cur)
        assert got == S.select(want, bounds, hyst, x, cur, oom)
        assert not oom[got[0]][S.bucket_of(bounds, x)], "selected an OOM configuration"
        cur = got[0]
    p.destroy()


@pytest.mark.gpu
def test_plan_mean_length_is_the_observed_average():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    earl = _lib()
    from paper_2510_05943_b200 import workloads as W
    from paper_2510_05943_b200.dispatch import EmulatedDispatch
    lens = W.c2_lengths(3).tolist()
    ed = EmulatedDispatch(8)
    plan = ed.plan(W.rollout_layout(len(lens), 8), W.layout(dp=2, tp=4), lens, W.field_set("tiny3"))
    assert plan.mean_length() == pytest.approx(S.observe(lens), rel=1e-12)
    p = earl.Policy(TP, BOUNDS, FIG3, hysteresis_tokens=500)
    assert p.select(plan.mean_length(), 0) == S.select(S.build_policy(TP, BOUNDS, FIG3), BOUNDS, 500,
                                                        S.observe(lens), 0)
