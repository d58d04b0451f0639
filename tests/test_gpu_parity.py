"""GPU parity: libearl_dispatch.so (called through the C ABI) against the CPU oracle.

Bit-exact on every byte of every destination rank, on the destination metadata (cu_seqlens,
seq_ids, tok_start), on the canonical plan table and on the byte accounting.  Payloads are
random bits (no float path can hide), receive buffers have 0xA5 guard bands on both sides.
"""
import random

import numpy as np
import pytest

from oracle import earl_oracle as O
from paper_2510_05943_b200 import workloads as W
from tests.helpers import random_layout, run_gpu_case

pytestmark = pytest.mark.gpu

GOLD_LENS = W.TINY_LENGTHS.tolist()
ODD_FIELDS = [("a", 4, 1, "x"), ("m", 1, 1, "x"), ("b", 2, 1, "x"), ("c", 1, 3, "x"),
              ("h", 2, 8, "x"), ("w", 2, 7, "x")]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2510_05943_b200 import build
    build.build()


@pytest.mark.parametrize("mode", ["exec", "stage"])
def test_c1_tiny_dp2_to_dp1(mode):
    src = W.rollout_layout(8, 2)
    dst = W.layout(dp=1, assign="contig")
    st = run_gpu_case(src, dst, GOLD_LENS, W.field_set("tiny3"), 2, mode=mode)
    assert st["moved"] == 1368 and st["total"] == 2508  # tests/golden/c1_tiny.json


@pytest.mark.parametrize("dst", [
    dict(dp=2, assign="contig"), dict(dp=2, assign="lpt"), dict(dp=1, sp=2, assign="contig"),
    dict(dp=1, tp=2, assign="contig"), dict(dp=2, assign="explicit", group_of_seq=[1, 0] * 4),
])
def test_c1_variants(dst):
    run_gpu_case(W.rollout_layout(8, 2), W.layout(**dst), GOLD_LENS, W.field_set("tiny3"), 2)


@pytest.mark.parametrize("seed", range(60))
def test_random_layouts(seed):
    rng = random.Random(seed)
    world = rng.randint(1, 8)
    n = rng.choice([0, 1, 3, rng.randint(0, 40), rng.randint(40, 300)])
    lens = [rng.choice([0, 1, 2, 15, 16, 17, rng.randint(0, 200), rng.randint(0, 3000)])
            for _ in range(n)]
    src = random_layout(rng, world, n)
    dst = random_layout(rng, world, n)
    fields = rng.sample(ODD_FIELDS, rng.randint(1, len(ODD_FIELDS)))
    run_gpu_case(src, dst, lens, fields, world, mode=rng.choice(["exec", "stage"]), seed=seed)


@pytest.mark.parametrize("mode", ["exec", "stage"])
@pytest.mark.parametrize("seed", range(6))
def test_host_pinned_sources_zero_copy(seed, mode):
    """Source arrays in pinned host memory (UVA): the copy kernel's TMA loads read them over
    PCIe, no separate H2D copy; the result is the same bytes."""
    rng = random.Random(100 + seed)
    world = rng.randint(2, 8)
    n = rng.randint(1, 200)
    lens = [rng.choice([0, 1, 17, rng.randint(0, 500)]) for _ in range(n)]
    src = random_layout(rng, world, n)
    dst = random_layout(rng, world, n)
    fields = rng.sample(ODD_FIELDS, rng.randint(1, len(ODD_FIELDS)))
    run_gpu_case(src, dst, lens, fields, world, mode=mode, seed=seed, host_src=True)


@pytest.mark.parametrize("seed", range(8))
def test_exec_per_source_rank(seed):
    """earl_dispatch_exec_src for every source rank, in a random order, equals one exec."""
    rng = random.Random(200 + seed)
    world = rng.randint(1, 8)
    n = rng.randint(0, 150)
    lens = [rng.choice([0, 1, 17, rng.randint(0, 700)]) for _ in range(n)]
    src = random_layout(rng, world, n)
    dst = random_layout(rng, world, n)
    fields = rng.sample(ODD_FIELDS, rng.randint(1, len(ODD_FIELDS)))
    run_gpu_case(src, dst, lens, fields, world, mode="exec_src", seed=seed,
                 host_src=seed % 2 == 1)


def test_plan_hash_is_a_function_of_the_inputs():
    """earl_plan_hash (the replicated-planning check): equal inputs, equal hashes -- also after a
    replan to other lengths and back; other lengths or layouts, other hashes."""
    import torch
    from paper_2510_05943_b200.dispatch import EmulatedDispatch
    lens = W.c2_lengths(0)[:200].tolist()
    src, dst = W.config_layouts("c3", 8, len(lens))
    ed = EmulatedDispatch(8)
    f = W.field_set("scalar6-fp32")
    a, b = ed.plan(src, dst, lens, f), ed.plan(src, dst, lens, f)
    h = a.hash()
    assert h == b.hash()
    other = list(lens)
    other[7] += 1
    c = ed.plan(src, dst, other, f)
    assert c.hash() != h
    d = ed.plan(src, W.layout(dp=4, tp=2, assign="contig"), lens, f)
    assert d.hash() != h
    a.replan(torch.as_tensor(np.asarray(other, dtype=np.int32)).cuda())
    assert a.hash() == c.hash()
    a.replan(torch.as_tensor(np.asarray(lens, dtype=np.int32)).cuda())
    assert a.hash() == h
    for p in (a, b, c, d):
        p.destroy()


def test_exec_src_rank_out_of_range():
    from paper_2510_05943_b200.dispatch import EmulatedDispatch
    from paper_2510_05943_b200.earl import EarlError
    ed = EmulatedDispatch(2)
    plan = ed.plan(W.rollout_layout(8, 2), W.layout(dp=1, assign="contig"), GOLD_LENS,
                   W.field_set("tiny3"))
    for bad in (-1, 2):
        with pytest.raises(EarlError):
            plan.exec_src(bad, [None] * 6, [None] * 6)
    plan.destroy()


def test_spec_acceptance_500_random_layout_pairs():
    """SPEC.md acceptance #4 (500 randomized layout pairs, bitwise equal to the oracle) scaled to
    tokens: every byte, the metadata and the canonical plan table of each case."""
    from paper_2510_05943_b200.dispatch import EmulatedDispatch
    rng = random.Random(4)
    eds = {}
    for case in range(500):
        world = rng.randint(1, 8)
        n = rng.randint(0, 60)
        lens = [rng.choice([0, 1, 5, rng.randint(0, 200)]) for _ in range(n)]
        src = random_layout(rng, world, n)
        dst = random_layout(rng, world, n)
        fields = rng.sample(ODD_FIELDS, rng.randint(1, 3))
        ed = eds.setdefault(world, EmulatedDispatch(world))
        run_gpu_case(src, dst, lens, fields, world, mode=rng.choice(["exec", "stage", "exec_src"]),
                     seed=1000 + case, ed=ed, guard=32)


@pytest.mark.parametrize("n_gpus", [2, 4, 8])
def test_c3_layouts_scalar6(n_gpus):
    """Config 3 shape (DPn -> DP max(1,n/4) x TP min(4,n)) on a 128-sequence slice of config 2."""
    lens = W.c2_lengths(0)[:128].tolist()
    src, dst = W.config_layouts("c3", n_gpus, len(lens))
    run_gpu_case(src, dst, lens, W.field_set("scalar6-fp32"), n_gpus, seed=n_gpus)


@pytest.mark.parametrize("n_gpus", [2, 4, 8])
def test_c4_layouts_sp2(n_gpus):
    """Config 4 shape (DPn -> DP n/2 x SP2) on 24 long sequences (4K-32K)."""
    lens = W.c4_lengths(0)[:24].tolist()
    src, dst = W.config_layouts("c4", n_gpus, len(lens))
    run_gpu_case(src, dst, lens, W.field_set("scalar6-bf16"), n_gpus, seed=10 + n_gpus,
                 mode="stage" if n_gpus == 4 else "exec")


@pytest.mark.parametrize("mode", ["exec", "stage"])
def test_alignment_every_residue_pair(mode):
    """SURVEY.md §4 copy-core fuzz: 1-byte field pieces of 0-1100 B whose source and destination
    offsets cover every (src mod 16, dst mod 16) pair (asserted on the oracle's table), so
    every realignment shift, head and tail of the copy engine runs against the oracle."""
    rng = random.Random(16)
    n = 2500
    lens = [rng.randint(0, 1100) for _ in range(n)]
    src = W.layout(dp=2, assign="given_counts", counts=[n // 2, n - n // 2])
    dst = W.layout(dp=3, assign="explicit", group_of_seq=[rng.randrange(3) for _ in range(n)])
    segs = O.route(src, dst, lens, 3)
    pairs = {(r[5] % 16, r[6] % 16) for r in segs if r[4] > r[3]}
    assert len(pairs) == 256, len(pairs)
    run_gpu_case(src, dst, lens, [("b", 1, 1, "x"), ("t", 1, 3, "x")], 3, mode=mode, seed=16)


def test_c2_full_scalar6_exec_and_stage():
    """BASELINE.json configs[1] at full size (512 episodes) with the scalar6 fields, 8-rank
    emulation of rollout DP8 -> train DP2 x TP4, element by element against the oracle."""
    lens = W.c2_lengths(0).tolist()
    src, dst = W.config_layouts("c2", 8, len(lens))
    run_gpu_case(src, dst, lens, W.field_set("scalar6-fp32"), 8, mode="exec", seed=1)
    run_gpu_case(src, dst, lens, W.field_set("scalar6-fp32"), 8, mode="stage", seed=2)


def test_c2_lpt_rebalance():
    lens = W.c2_lengths(0).tolist()
    src, dst = W.config_layouts("c2-lpt", 8, len(lens))
    run_gpu_case(src, dst, lens, W.field_set("scalar6-bf16"), 8, seed=3)


def test_lpt_max_size_groups_match_oracle():
    """LPT at its maximum N (8192): the plan (hence g(i)) equals the oracle's."""
    rng = np.random.default_rng(4)
    lens = rng.integers(0, 5000, size=8192).tolist()
    src = W.rollout_layout(8192, 8)
    dst = W.layout(dp=8, assign="lpt")
    run_gpu_case(src, dst, lens, [("m", 1, 1, "x")], 8, seed=4)


def test_uniform_sweep_round_robin():
    """Config 5 shape: DP8 -> EXPLICIT round-robin (uniform all-to-allv)."""
    lens = [4096] * 64
    src, dst = W.config_layouts("c5", 8, len(lens))
    run_gpu_case(src, dst, lens, W.field_set("scalar6-fp32"), 8, seed=5)


def test_alignment_fuzz_many_short_sequences():
    """Every (src mod 16, dst mod 16) combination: 1-byte and odd-width fields over many
    sequences of lengths 0..40 regrouped with LPT (scrambles offsets on both sides)."""
    rng = np.random.default_rng(6)
    lens = rng.integers(0, 41, size=700).tolist()
    src = W.layout(dp=3, sp=2, assign="contig")
    dst = W.layout(rank0=1, dp=5, tp=1, assign="lpt")
    run_gpu_case(src, dst, lens, [("m", 1, 1, "x"), ("c", 1, 3, "x"), ("w", 2, 7, "x")], 7,
                 seed=6, mode="exec")
    run_gpu_case(src, dst, lens, [("m", 1, 1, "x"), ("c", 1, 3, "x"), ("w", 2, 7, "x")], 7,
                 seed=7, mode="stage")


def test_round_trip_identity_on_gpu():
    import torch
    from paper_2510_05943_b200.dispatch import EmulatedDispatch
    lens = W.c2_lengths(1)[:96].tolist()
    fields = W.field_set("scalar6-fp32")
    src = W.rollout_layout(96, 8)
    dst = W.layout(dp=2, sp=2, tp=2, assign="contig")
    glob = W.gen_global_fields(fields, sum(lens), random_bits=True)
    src_arrays = O.rank_arrays_from_global(src, lens, O.assign_groups(src, lens), glob, fields)
    ed = EmulatedDispatch(8)
    p1 = ed.plan(src, dst, lens, fields)
    send = [torch.from_numpy(src_arrays[r][f]).cuda() for r in range(8) for f in range(6)]
    mid = ed.alloc_recv(p1, fields)
    p1.exec(send, ed.flat(mid))
    inv_src, inv_dst = O.inverse_layouts(src, dst, lens)
    p2 = ed.plan(inv_src, inv_dst, lens, fields)
    back = ed.alloc_recv(p2, fields)
    p2.exec(ed.flat(mid), ed.flat(back))
    torch.cuda.synchronize()
    for r in range(8):
        for f in range(6):
            assert np.array_equal(back[r][f].cpu().numpy(), src_arrays[r][f])


def test_plan_is_deterministic():
    from paper_2510_05943_b200.dispatch import EmulatedDispatch
    lens = W.c4_lengths(2).tolist()
    ed = EmulatedDispatch(8)
    src, dst = W.config_layouts("c4", 8, len(lens))
    f = W.field_set("scalar6-fp32")
    a = ed.plan(src, dst, lens, f).export()
    b = ed.plan(src, dst, lens, f).export()
    assert a == b == O.route(src, dst, lens, 8)


# ---------------------------------------------------------------------------------------
# errors
# ---------------------------------------------------------------------------------------

def test_device_latched_errors():
    from paper_2510_05943_b200.dispatch import EmulatedDispatch
    from paper_2510_05943_b200.earl import EarlError
    ed = EmulatedDispatch(2)
    f = W.field_set("tiny3")
    p = ed.plan(W.layout(dp=1), W.layout(dp=2), [3, -1, 2], f)
    with pytest.raises(EarlError) as e:
        p.local_sizes(0)
    assert e.value.name == "EARL_ERR_INVALID_ARGUMENT"
    p = ed.plan(W.layout(dp=1), W.layout(dp=2, assign="explicit", group_of_seq=[0, 5, 1]),
                [3, 1, 2], f)
    with pytest.raises(EarlError) as e:
        p.stats()
    assert e.value.name == "EARL_ERR_LAYOUT"


EDGE = 2**31 - 1
CAPACITY_CASES = [
    (dict(dp=1, assign="contig"), [2**30, 2**30 - 1]),           # exactly INT32_MAX: fits
    (dict(dp=1, assign="contig"), [2**30, 2**30]),               # one token over
    (dict(dp=1, assign="contig"), [2**20] * 2049),               # 2^31 + 2^20
    (dict(dp=1, sp=2, assign="contig"), [EDGE, EDGE - 2]),       # SP rank 0 at the edge
    (dict(dp=1, sp=2, assign="contig"), [EDGE, EDGE]),           # SP rank 0 over
    (dict(dp=2, assign="explicit", group_of_seq=[0, 0, 1]), [2**30, 2**30, 5]),  # partitioned path
    (dict(dp=2, assign="explicit", group_of_seq=[0, 1, 1]), [2**30, 2**30, 5]),
    (dict(dp=2, tp=2, assign="contig"), [2**30, 2**30]),         # two groups of 2^30: fit
]


@pytest.mark.parametrize("k", range(len(CAPACITY_CASES)))
def test_planner_capacity_latch_matches_oracle(k):
    """Reading c12 (int32 cu_seqlens): the planner's device latch fires exactly when the oracle's
    check_capacity does -- lengths only, no payload (a plan of > 2^31 tokens moves nothing)."""
    from paper_2510_05943_b200.dispatch import EmulatedDispatch
    from paper_2510_05943_b200.earl import EarlError
    dst_d, lens = CAPACITY_CASES[k]
    dst = W.layout(**dst_d)
    src = W.rollout_layout(len(lens), 2)
    try:
        O.check_capacity(dst, lens, O.assign_groups(dst, lens))
        want_err = False
    except O.OracleError as e:
        assert e.code == O.ERR_CAPACITY
        want_err = True
    ed = EmulatedDispatch(4)
    plan = ed.plan(src, dst, lens, W.field_set("tiny3"))
    if want_err:
        with pytest.raises(EarlError) as e:
            plan.sync()
        assert e.value.name == "EARL_ERR_CAPACITY"
        assert "INT32_MAX" in str(e.value)
    else:
        plan.sync()
        hd = O.holdings(dst, lens, O.assign_groups(dst, lens))
        for r, h in hd.items():
            assert plan.local_sizes(r)[1] == h["n_tokens"]
    plan.destroy()


@pytest.mark.parametrize("bad,name", [
    (dict(dp=3), "EARL_ERR_LAYOUT"),
    (dict(dp=2, assign="given_counts", counts=[1, 1]), "EARL_ERR_LAYOUT"),
    (dict(rank0=1, dp=2), "EARL_ERR_LAYOUT"),
])
def test_host_layout_errors(bad, name):
    from paper_2510_05943_b200.dispatch import EmulatedDispatch
    from paper_2510_05943_b200.earl import EarlError
    ed = EmulatedDispatch(2)
    with pytest.raises(EarlError) as e:
        ed.plan(W.layout(dp=1), W.layout(**bad), [3, 1, 2, 5], W.field_set("tiny3"))
    assert e.value.name == name


def test_lpt_capacity_and_misaligned_buffers():
    import torch
    from paper_2510_05943_b200.dispatch import EmulatedDispatch
    from paper_2510_05943_b200.earl import EarlError
    ed = EmulatedDispatch(2)
    with pytest.raises(EarlError) as e:
        ed.plan(W.layout(dp=1), W.layout(dp=2, assign="lpt"), [1] * 8193, W.field_set("tiny3"))
    assert e.value.name == "EARL_ERR_CAPACITY"
    f = [("a", 4, 1, "x")]
    p = ed.plan(W.layout(dp=1), W.layout(dp=2), [4, 4], f)
    buf = torch.zeros(64, dtype=torch.uint8, device="cuda")
    with pytest.raises(EarlError) as e:
        p.exec([buf[4:], None], [buf[16:], buf[32:]])
    assert e.value.name == "EARL_ERR_INVALID_ARGUMENT"


@pytest.mark.parametrize("n,dst", [
    (60000, dict(dp=2, sp=2, tp=2, assign="contig")),
    (100000, dict(dp=8, assign="explicit", group_of_seq=None)),
    (45000, dict(rank0=1, dp=3, sp=2, assign="given_counts")),
])
def test_large_n_cooperative_planner(n, dst):
    """N large enough for a multi-CTA cooperative planner grid (G = ceil(N/4096) > 1): plan,
    bytes and metadata equal the oracle's."""
    rng = np.random.default_rng(n)
    lens = rng.integers(0, 48, size=n).tolist()
    dst = dict(dst)
    if dst["assign"] == "explicit":
        dst["group_of_seq"] = rng.integers(0, dst["dp"], size=n).astype(np.int32)
    if dst["assign"] == "given_counts":
        dst["counts"] = W.near_equal_counts(n, dst["dp"])
    run_gpu_case(W.rollout_layout(n, 8), W.layout(**dst), lens, [("m", 1, 1, "x"), ("a", 4, 1, "x")],
                 8, seed=9)


def test_plan_outlives_comm_handle():
    """Plans hold a reference on their comm: destroying the comm handle first (as a garbage
    collector may) leaves the plan usable and the device error state clean."""
    import torch
    from paper_2510_05943_b200.dispatch import EmulatedDispatch
    ed = EmulatedDispatch(2)
    f = [("a", 4, 1, "x")]
    p = ed.plan(W.layout(dp=1), W.layout(dp=2), [4, 4], f)
    recv = ed.alloc_recv(p, f)
    ed.comm.destroy()
    src = torch.arange(8, dtype=torch.int32, device="cuda").view(torch.uint8)
    p.exec([src, None], ed.flat(recv))
    torch.cuda.synchronize()
    p.sync()
    assert recv[0][0].view(torch.int32).tolist() == [0, 1, 2, 3]
    assert recv[1][0].view(torch.int32).tolist() == [4, 5, 6, 7]
    p.destroy()


_GRID_SCRIPT = r"""
import hashlib, sys, numpy as np, torch
sys.path.insert(0, {root!r})
from oracle import earl_oracle as O
from paper_2510_05943_b200 import workloads as W
from paper_2510_05943_b200.dispatch import EmulatedDispatch
rng = np.random.default_rng(21)
n = 20000
lens = rng.integers(0, 60, size=n).tolist()
out = []
for dst in (W.layout(dp=2, sp=2, tp=2, assign="contig"),
            W.layout(dp=4, assign="lpt") if False else W.layout(dp=4, sp=2, assign="explicit",
                     group_of_seq=rng.integers(0, 4, size=n).astype(np.int32))):
    ed = EmulatedDispatch(8)
    fields = [("m", 1, 1, "x"), ("a", 4, 1, "x")]
    p = ed.plan(W.rollout_layout(n, 8), dst, lens, fields)
    segs = p.export()
    h = hashlib.blake2b(np.asarray(segs, dtype=np.int64).tobytes(), digest_size=16).hexdigest()
    st = p.stats()
    out.append(h + ":" + str(st["records"]) + ":" + str(st["total"]))
print("|".join(out))
"""


def test_plan_independent_of_planner_grid():
    """The cooperative planner's result does not depend on its grid size: G = 1, 3, 7 and the
    automatic choice give byte-identical canonical plans (subprocesses: EARL_PLAN_GRID is read
    once per process)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = _GRID_SCRIPT.format(root=root)
    outs = {}
    for g in ("1", "3", "7", ""):
        env = dict(os.environ)
        if g:
            env["EARL_PLAN_GRID"] = g
        else:
            env.pop("EARL_PLAN_GRID", None)
        r = subprocess.run([sys.executable, "-c", script], capture_output=True, text=True, env=env,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs[g] = r.stdout.strip().splitlines()[-1]
    assert len(set(outs.values())) == 1, outs


# ---------------------------------------------------------------------------------------
# SP split variants (readings n1 zigzag, n2 flat, n3 threshold)
# ---------------------------------------------------------------------------------------

@pytest.mark.parametrize("split,extra", [("zigzag", {}), ("flat", {}),
                                         ("threshold", {"sp_min_len": 20})])
def test_golden_sp_variants_on_gpu(split, extra):
    dst = W.layout(dp=1, sp=2, assign="contig", sp_split=split, **extra)
    run_gpu_case(W.rollout_layout(8, 2), dst, GOLD_LENS, W.field_set("tiny3"), 2)


@pytest.mark.parametrize("split", ["zigzag", "flat", "threshold"])
@pytest.mark.parametrize("n_gpus", [4, 8])
def test_c4_sp_variants(split, n_gpus):
    """Config 4's DPn -> DP n/2 x SP2 with each split rule (threshold: split sequences >= 8K)."""
    lens = W.c4_lengths(0)[:24].tolist()
    src, dst = W.config_layouts("c4", n_gpus, len(lens))
    dst = dict(dst, sp_split=split, sp_min_len=8192 if split == "threshold" else 0)
    run_gpu_case(src, dst, lens, W.field_set("scalar6-bf16"), n_gpus, seed=30 + n_gpus,
                 mode="stage" if split == "flat" else "exec")


@pytest.mark.parametrize("seed", range(40))
def test_random_variant_layouts_on_gpu(seed):
    from tests.test_oracle_sp_variants import with_split
    rng = random.Random(5000 + seed)
    world = rng.randint(1, 8)
    n = rng.choice([0, 1, 5, rng.randint(0, 60), rng.randint(60, 250)])
    lens = [rng.choice([0, 1, 2, 7, rng.randint(0, 100), rng.randint(0, 1500)]) for _ in range(n)]
    src = with_split(rng, random_layout(rng, world, n))
    dst = with_split(rng, random_layout(rng, world, n))
    fields = rng.sample(ODD_FIELDS, rng.randint(1, 4))
    run_gpu_case(src, dst, lens, fields, world, mode=rng.choice(["exec", "stage"]), seed=seed)


def test_large_n_variants_cooperative():
    rng = np.random.default_rng(77)
    n = 30000
    lens = rng.integers(0, 40, size=n).tolist()
    for dst in (W.layout(dp=2, sp=4, assign="contig", sp_split="zigzag"),
                W.layout(dp=4, sp=2, assign="contig", sp_split="flat"),
                W.layout(dp=2, sp=2, tp=2, assign="contig", sp_split="threshold", sp_min_len=20)):
        run_gpu_case(W.rollout_layout(n, 8), dst, lens, [("m", 1, 1, "x")], 8, seed=11)


# ---------------------------------------------------------------------------------------
# plan reuse and CUDA graphs
# ---------------------------------------------------------------------------------------

def _fill_and_expect(src, dst, lens, fields, world, cap_tok, dev, seed):
    """Source buffers (capacity cap_tok tokens per rank) filled for `lens`, and the oracle."""
    import torch
    glob = W.gen_global_fields(fields, sum(lens), seed_base=seed, random_bits=True)
    src_arrays = O.rank_arrays_from_global(src, lens, O.assign_groups(src, lens), glob, fields)
    want, meta, segs = O.dispatch(src, dst, lens, src_arrays, fields, world)
    return src_arrays, want, segs


def test_replan_and_cuda_graph_replay():
    import torch
    from paper_2510_05943_b200.dispatch import EmulatedDispatch
    world, n = 8, 200
    fields = [("a", 4, 1, "x"), ("m", 1, 1, "x"), ("h", 2, 16, "x")]
    Bf = O.field_bytes(fields)
    rng = np.random.default_rng(3)
    batches = [rng.integers(0, 400, size=n).tolist() for _ in range(4)]
    src = W.rollout_layout(n, world)
    dst = W.layout(dp=2, sp=2, tp=2, assign="contig", sp_split="zigzag")
    cap = max(sum(b) for b in batches)
    ed = EmulatedDispatch(world)
    dev = ed.device
    send = [torch.zeros(cap * b, dtype=torch.uint8, device=dev) for _ in range(world) for b in Bf]
    recv = [torch.zeros(cap * b, dtype=torch.uint8, device=dev) for _ in range(world) for b in Bf]
    lens_dev = torch.tensor(batches[0], dtype=torch.int32, device=dev)
    plan = ed.plan(src, dst, lens_dev, fields)

    def load(lens, seed):
        src_arrays, want, segs = _fill_and_expect(src, dst, lens, fields, world, cap, dev, seed)
        for r in range(world):
            for f in range(len(fields)):
                a = src_arrays[r][f]
                if a.size:
                    send[r * len(fields) + f][: a.size].copy_(torch.from_numpy(a))
        return want, segs

    def check(want):
        for r, arrs in want.items():
            for f in range(len(fields)):
                got = recv[r * len(fields) + f][: arrs[f].size].cpu().numpy()
                assert np.array_equal(got, arrs[f]), (r, f)

    # 1) replan: new lengths into the same plan memory
    want, segs = load(batches[1], 11)
    lens_dev.copy_(torch.tensor(batches[1], dtype=torch.int32))
    plan.replan(lens_dev)
    assert plan.export() == segs
    plan.exec(send, recv)
    torch.cuda.synchronize()
    check(want)
    # 2) capture replan + exec in a CUDA graph, replay for two more batches
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        plan.replan(lens_dev, stream=s)
        plan.exec(send, recv, stream=s)
    for k, lens in enumerate(batches[2:]):
        want, segs = load(lens, 20 + k)
        lens_dev.copy_(torch.tensor(lens, dtype=torch.int32))
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        check(want)
        assert plan.export() == segs


# ---------------------------------------------------------------------------------------
# NEXT-2: per-sequence fields routed with their sequences (reading n4)
# ---------------------------------------------------------------------------------------

@pytest.mark.parametrize("seed", range(20))
def test_seq_fields_on_gpu(seed):
    import torch
    from paper_2510_05943_b200.dispatch import EmulatedDispatch, plan_seq_fields
    from tests.test_oracle_sp_variants import with_split
    rng = random.Random(7000 + seed)
    world = rng.randint(1, 8)
    n = rng.choice([0, 1, rng.randint(1, 40), rng.randint(40, 400)])
    lens = [rng.randint(0, 500) for _ in range(n)]
    src = with_split(rng, random_layout(rng, world, n))
    dst = with_split(rng, random_layout(rng, world, n))
    sf = [("reward", 4, 1, "x"), ("score", 2, 3, "x")]
    Bs = O.field_bytes(sf)
    gs = O.assign_groups(src, lens)
    hs = O.seq_holdings(src, lens, gs)
    glob = [np.random.default_rng(seed * 3 + f).integers(0, 256, size=n * Bs[f], dtype=np.uint8)
            for f in range(len(sf))]
    src_arrays = {r: [np.concatenate([glob[f][i * Bs[f]:(i + 1) * Bs[f]] for i in m])
                      if m else np.zeros(0, dtype=np.uint8) for f in range(len(sf))]
                  for r, m in hs.items()}
    want = O.dispatch_seq_fields(src, dst, lens, src_arrays, sf, world)
    ed = EmulatedDispatch(world)
    tp = ed.plan(src, dst, lens, W.field_set("tiny3"))
    sp = plan_seq_fields(ed.comm, tp, ed._src, ed._dst, sf, ed.device)
    st = sp.stats()
    send = [torch.from_numpy(src_arrays[r][f]).cuda() if r in src_arrays and src_arrays[r][f].size
            else None for r in range(world) for f in range(len(sf))]
    recv = [torch.zeros(max(1, int(st["n_local_tokens"][r]) * Bs[f]), dtype=torch.uint8, device="cuda")
            for r in range(world) for f in range(len(sf))]
    sp.exec(send, recv)
    torch.cuda.synchronize()
    for d, arrs in want.items():
        for f in range(len(sf)):
            got = recv[d * len(sf) + f][: arrs[f].size].cpu().numpy()
            assert np.array_equal(got, arrs[f]), (d, f)
    # the token plan re-planned for other lengths (same N): the per-sequence plan follows it
    # (earl_plan_replan on it re-reads the token plan's groups on the device)
    if n and seed % 2 == 0:
        lens2 = [rng.randint(0, 500) for _ in range(n)]
        want2 = O.dispatch_seq_fields(src, dst, lens2, {
            r: [np.concatenate([glob[f][i * Bs[f]:(i + 1) * Bs[f]] for i in m])
                if m else np.zeros(0, dtype=np.uint8) for f in range(len(sf))]
            for r, m in O.seq_holdings(src, lens2, O.assign_groups(src, lens2)).items()}, sf, world)
        if all(O.seq_holdings(src, lens2, O.assign_groups(src, lens2)).get(r) == hs.get(r)
               for r in range(world)):
            tp.replan(torch.as_tensor(np.asarray(lens2, dtype=np.int32)).cuda())
            sp.replan()
            st2 = sp.stats()
            recv2 = [torch.zeros(max(1, int(st2["n_local_tokens"][r]) * Bs[f]), dtype=torch.uint8,
                                 device="cuda") for r in range(world) for f in range(len(sf))]
            sp.exec(send, recv2)
            torch.cuda.synchronize()
            for d, arrs in want2.items():
                for f in range(len(sf)):
                    got = recv2[d * len(sf) + f][: arrs[f].size].cpu().numpy()
                    assert np.array_equal(got, arrs[f]), ("replan", d, f)
    tp.destroy()   # the per-sequence plan keeps its token plan alive
    sp.exec(send, recv)
    torch.cuda.synchronize()
    sp.destroy()


@pytest.mark.parametrize("gamma", [1.0, 0.97, 0.0])
@pytest.mark.parametrize("tp", [1, 2])
@pytest.mark.parametrize("kernel", ["units", "windows", "coop", "auto"])
def test_distributed_advantages_on_gpu(gamma, tp, kernel, monkeypatch):
    """Reading n5 on the GPU (fp32 tokens, fp64 statistics) against the fp64 oracle, with every
    returns kernel forced (the cooperative, the single-pass unit and the windowed look-back
    kernel) and with the device's own choice (auto: all three launched, gated on the header).
    Tolerance: the fp32 recurrence G_t = v_t + gamma G_{t+1} accumulates at most
    u * min(L, 1/(1-gamma)) * max|G| rounding error (u = 2^-24), times 4 for the warp-parallel
    composition; A inherits it divided by sigma."""
    import torch
    from paper_2510_05943_b200.dispatch import EmulatedDispatch
    if kernel != "auto":  # auto: the plan is not synchronised, every kernel launches gated
        monkeypatch.setenv("EARL_RETURNS", kernel)
    rng = np.random.default_rng(int(gamma * 100) + tp)
    world = 8
    n = 300
    lens = W.lognormal_lengths(n, 600, 0.8, 1, 3000, seed=5).tolist()
    lens[3] = 0
    src = W.layout(dp=world // tp, tp=tp, assign="contig")
    T = sum(lens)
    glob_r = rng.standard_normal(T).astype(np.float32)
    glob_m = (rng.random(T) < 0.75).astype(np.uint8)
    fr = [("r", 4, 1, "x"), ("m", 1, 1, "x")]
    arrs = O.rank_arrays_from_global(src, lens, O.assign_groups(src, lens),
                                     [glob_r.view(np.uint8), glob_m], fr)
    rewards = {k: v[0].view(np.float32) for k, v in arrs.items()}
    masks = {k: v[1] for k, v in arrs.items()}
    G, A, R, stats = O.distributed_advantages(src, lens, rewards, masks, gamma, 1e-8, world)

    ed = EmulatedDispatch(world)
    plan = ed.plan(src, W.layout(dp=2, sp=2, tp=2, assign="contig"), lens, W.field_set("tiny3"))
    dev = ed.device
    d_r = [torch.from_numpy(rewards[r].copy()).to(dev) for r in range(world)]
    d_m = [torch.from_numpy(masks[r].copy()).to(dev) for r in range(world)]
    d_G = [torch.zeros(max(1, rewards[r].size), dtype=torch.float32, device=dev) for r in range(world)]
    d_A = [torch.zeros(max(1, rewards[r].size), dtype=torch.float32, device=dev) for r in range(world)]
    ns = plan.stats()["n_local_seqs"]
    d_R = [torch.zeros(max(1, len(R[r])), dtype=torch.float32, device=dev) for r in range(world)]
    partial = torch.zeros(3, dtype=torch.float64, device=dev)
    plan.returns(gamma, d_r, d_m, d_G, partial, seq_return=d_R)
    plan.advantages(partial, 1e-8, d_G, d_m, d_A)  # emulated: partials already cover the batch
    torch.cuda.synchronize()
    assert ns is not None
    Lmax = max(lens)
    horizon = Lmax if gamma >= 1.0 else min(Lmax, 1.0 / (1.0 - gamma))
    gmax = max(np.abs(G[r]).max() if G[r].size else 0 for r in G)
    atol_g = 4 * 2.0 ** -24 * horizon * gmax + 1e-6
    got_stats = partial.cpu().numpy()
    assert got_stats[0] == stats[0]
    assert np.allclose(got_stats[1:], stats[1:], rtol=1e-5, atol=atol_g * stats[0])
    sigma = np.sqrt(max(stats[2] / stats[0] - (stats[1] / stats[0]) ** 2, 0))
    for r in range(world):
        n_r = rewards[r].size
        assert np.allclose(d_G[r][:n_r].cpu().numpy(), G[r], rtol=0, atol=atol_g), r
        assert np.allclose(d_A[r][:n_r].cpu().numpy(), A[r], rtol=0, atol=atol_g / sigma + 1e-5), r
        assert np.allclose(d_R[r][: len(R[r])].cpu().numpy(), R[r], rtol=0, atol=atol_g), r


def test_returns_need_whole_sequences():
    from paper_2510_05943_b200.dispatch import EmulatedDispatch
    from paper_2510_05943_b200.earl import EarlError
    import torch
    ed = EmulatedDispatch(2)
    plan = ed.plan(W.layout(dp=1, sp=2), W.layout(dp=2), [4, 4], W.field_set("tiny3"))
    p = torch.zeros(3, dtype=torch.float64, device="cuda")
    with pytest.raises(EarlError) as e:
        plan.returns(1.0, [None, None], [None, None], [None, None], p)
    assert e.value.name == "EARL_ERR_UNSUPPORTED"


def _adv_case(lens, src, gamma, world, shift=0, repeats=1, graph=False, seed=0):
    """Run earl_returns + earl_advantages (emulated comm) and compare with the fp64 oracle.
    shift > 0 offsets every device buffer by `shift` elements (the unaligned scalar path)."""
    import torch
    from paper_2510_05943_b200.dispatch import EmulatedDispatch
    rng = np.random.default_rng(seed)
    T = sum(lens)
    glob_r = rng.standard_normal(T).astype(np.float32)
    glob_m = (rng.random(T) < 0.75).astype(np.uint8)
    fr = [("r", 4, 1, "x"), ("m", 1, 1, "x")]
    arrs = O.rank_arrays_from_global(src, lens, O.assign_groups(src, lens),
                                     [glob_r.view(np.uint8), glob_m], fr)
    rewards = {k: v[0].view(np.float32) for k, v in arrs.items()}
    masks = {k: v[1] for k, v in arrs.items()}
    G, A, R, stats = O.distributed_advantages(src, lens, rewards, masks, gamma, 1e-8, world)
    ed = EmulatedDispatch(world)
    plan = ed.plan(src, W.layout(dp=1, assign="contig"), lens, W.field_set("tiny3"))
    dev = ed.device

    def buf(host, dtype):
        t = torch.zeros(host.size + shift + 4, dtype=dtype, device=dev)
        t[shift:shift + host.size] = torch.from_numpy(host.copy()).to(dev)
        return t[shift:]
    empty_f = np.zeros(0, np.float32)
    d_r = [buf(rewards.get(r, empty_f), torch.float32) for r in range(world)]
    d_m = [buf(masks.get(r, np.zeros(0, np.uint8)), torch.uint8) for r in range(world)]
    d_G = [buf(np.full(rewards.get(r, empty_f).size, np.nan, np.float32), torch.float32) for r in range(world)]
    d_A = [buf(np.full(rewards.get(r, empty_f).size, np.nan, np.float32), torch.float32) for r in range(world)]
    d_R = [buf(np.full(len(R.get(r, [])), np.nan, np.float32), torch.float32) for r in range(world)]
    partial = torch.zeros(3, dtype=torch.float64, device=dev)

    def step():
        partial.zero_()
        plan.returns(gamma, d_r, d_m, d_G, partial, seq_return=d_R)
        plan.advantages(partial, 1e-8, d_G, d_m, d_A)
    step()  # allocates the workspace outside any capture
    if graph:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            partial.zero_()
            plan.returns(gamma, d_r, d_m, d_G, partial, seq_return=d_R,
                         stream=torch.cuda.current_stream().cuda_stream)
            plan.advantages(partial, 1e-8, d_G, d_m, d_A,
                            stream=torch.cuda.current_stream().cuda_stream)
        for x in d_G + d_A + d_R:
            x.fill_(float("nan"))
        for _ in range(repeats):
            g.replay()
    else:
        for _ in range(repeats - 1):
            step()
    torch.cuda.synchronize()
    plan.sync()
    Lmax = max(lens) if lens else 1
    horizon = Lmax if gamma >= 1.0 else min(Lmax, 1.0 / (1.0 - gamma))
    gmax = max([np.abs(G[r]).max() for r in G if G[r].size] + [1.0])
    atol_g = 4 * 2.0 ** -24 * horizon * gmax + 1e-6
    got = partial.cpu().numpy()
    assert got[0] == stats[0]
    assert np.allclose(got[1:], stats[1:], rtol=1e-5, atol=atol_g * max(stats[0], 1))
    sigma = np.sqrt(max(stats[2] / stats[0] - (stats[1] / stats[0]) ** 2, 0)) if stats[0] else 1.0
    for r in G:
        n_r = rewards[r].size
        assert np.allclose(d_G[r][:n_r].cpu().numpy(), G[r], rtol=0, atol=atol_g), r
        assert np.allclose(d_A[r][:n_r].cpu().numpy(), A[r], rtol=0, atol=atol_g / sigma + 1e-5), r
        assert np.allclose(d_R[r][:len(R[r])].cpu().numpy(), R[r], rtol=0, atol=atol_g), r
    plan.destroy()


ADV_EDGE_CASES = {
    # one 50K-token sequence: 49 windows chained through the look-back (gamma = 1: no decay)
    "one_long": ([50_000], 1),
    # lengths straddling the 1024-token window and the 4-token quad
    "window_edges": ([1023, 1024, 1025, 1, 2, 3, 4, 5, 2047, 2048, 2049, 128, 127, 129], 2),
    # zero-length sequences in the middle and at the end of a rank; a rank with only empties
    "zeros": ([0, 7, 0, 0, 1500, 0, 0, 0, 0, 3, 0, 0], 4),
    # thousands of 1..3-token sequences: many ends per window
    "tiny": ([1 + (i % 3) for i in range(5000)], 8),
}


@pytest.mark.parametrize("case", sorted(ADV_EDGE_CASES))
@pytest.mark.parametrize("gamma", [1.0, 0.9])
@pytest.mark.parametrize("shift", [0, 1])
@pytest.mark.parametrize("kernel", ["units", "windows", "coop", "auto"])
def test_returns_edge_cases(case, gamma, shift, kernel, monkeypatch):
    if kernel != "auto":  # auto: the plan is not synchronised, every kernel launches gated
        monkeypatch.setenv("EARL_RETURNS", kernel)
    lens, dp = ADV_EDGE_CASES[case]
    src = W.layout(dp=dp, assign="given_counts", counts=W.near_equal_counts(len(lens), dp))
    _adv_case(list(lens), src, gamma, 8, shift=shift, seed=len(lens))


@pytest.mark.parametrize("graph", [False, True])
@pytest.mark.parametrize("kernel", ["units", "windows", "coop", "auto"])
def test_returns_repeat_and_graph(graph, kernel, monkeypatch):
    """The look-back workspace / unit table is reused across launches and graph replays."""
    if kernel != "auto":  # auto: the plan is not synchronised, every kernel launches gated
        monkeypatch.setenv("EARL_RETURNS", kernel)
    lens = W.lognormal_lengths(200, 1500, 0.8, 1, 6000, seed=9).tolist()
    _adv_case(lens, W.layout(dp=4, tp=2, assign="lpt"), 0.99, 8, repeats=5, graph=graph)


def test_returns_source_rank_above_int32_tokens(monkeypatch):
    """Maximum size (reading n5): one source rank holding 2^31 + 2^20 tokens (2049 sequences of
    2^20 on DP1; the destination DP4 shards stay under INT32_MAX).  The unit kernel keeps rank
    positions in int32, so the automatic choice takes the windowed kernel (int64 positions): the
    returns of the sequences around token 2^31 equal the oracle's per-sequence recurrence, and the
    masked-token count is exact.  Forcing the unit kernel latches EARL_ERR_CAPACITY."""
    import torch
    from paper_2510_05943_b200.dispatch import EmulatedDispatch
    from paper_2510_05943_b200.earl import EarlError
    L, n = 2**20, 2049
    T = L * n
    free = torch.cuda.mem_get_info()[0]
    if free < 24 * 2**30:
        pytest.skip("needs ~20 GB of device memory")
    ed = EmulatedDispatch(4)
    plan = ed.plan(W.layout(dp=1), W.layout(dp=4, assign="contig"), [L] * n, W.field_set("tiny3"))
    plan.sync()
    gen = torch.Generator(device="cuda").manual_seed(11)
    r = torch.randn(T, device="cuda", generator=gen)
    m = (torch.rand(T, device="cuda", generator=gen) < 0.8).to(torch.uint8)
    G = torch.empty(T, device="cuda")
    dummy_f = torch.zeros(4, device="cuda")
    dummy_m = torch.zeros(4, dtype=torch.uint8, device="cuda")
    part = torch.zeros(3, dtype=torch.float64, device="cuda")
    gamma = 0.99
    plan.returns(gamma, [r, dummy_f, dummy_f, dummy_f], [m, dummy_m, dummy_m, dummy_m],
                 [G, dummy_f.clone(), dummy_f.clone(), dummy_f.clone()], part)
    torch.cuda.synchronize()
    plan.sync()
    assert part[0].item() == float(m.sum(dtype=torch.int64).item())
    atol = 4 * 2.0 ** -24 * (1.0 / (1.0 - gamma)) * 8.0 + 1e-6
    for p in (0, 2047, 2048):  # 2048 starts at token 2^31
        lo = p * L
        rr = r[lo:lo + L].cpu().numpy()
        mm = m[lo:lo + L].cpu().numpy()
        want = O.discounted_returns(rr, mm, gamma)
        gmax = max(1.0, float(np.abs(want).max()))
        got = G[lo:lo + L].cpu().numpy()
        assert np.allclose(got, want, rtol=0, atol=atol * gmax), p
    monkeypatch.setenv("EARL_RETURNS", "units")
    plan.returns(gamma, [r, dummy_f, dummy_f, dummy_f], [m, dummy_m, dummy_m, dummy_m],
                 [G, dummy_f.clone(), dummy_f.clone(), dummy_f.clone()], part)
    torch.cuda.synchronize()
    with pytest.raises(EarlError) as e:
        plan.sync()
    assert e.value.name == "EARL_ERR_CAPACITY"
    plan.destroy()
    del r, m, G
    torch.cuda.empty_cache()


@pytest.mark.parametrize("seed", range(40))
def test_sp1_fast_planner_equals_general_planner(seed, monkeypatch):
    """The SP = 1 single-pass planner (planner_sp1_kernel) and the general phased planner give
    the same plan, header tables and records included (earl_plan_hash), and the oracle's
    segment table -- for random SP = 1 layout pairs of every assignment rule, N up to 40K
    (multi-CTA grids), zero-length sequences and forced grid sizes."""
    import torch
    from paper_2510_05943_b200.dispatch import EmulatedDispatch
    rng = random.Random(9100 + seed)
    world = rng.randint(1, 8)
    n = rng.choice([0, 1, 7, rng.randint(1, 600), rng.randint(600, 5000), rng.randint(5000, 40000)])
    lens = [rng.choice([0, 1, rng.randint(0, 300), rng.randint(0, 9000)]) for _ in range(n)]

    def sp1(lay):
        lay = dict(lay, sp=1)
        if lay["assign"] == "lpt" and n > 8192:
            lay["assign"] = "contig"
        lay["sp_split"] = rng.choice(["block", "flat", "threshold"])
        lay["sp_min_len"] = rng.randint(0, 500)
        return lay

    src, dst = sp1(random_layout(rng, world, n)), sp1(random_layout(rng, world, n))
    if src["assign"] == "given_counts" and src["counts"] is None:
        src["counts"] = W.near_equal_counts(n, src["dp"])
    fields = [("a", 4, 1, "x"), ("b", 2, 3, "x")]
    ed = EmulatedDispatch(world)
    lens_dev = torch.as_tensor(np.asarray(lens, dtype=np.int32)).cuda()
    if seed % 4 == 3:
        monkeypatch.setenv("EARL_PLAN_GRID", str(rng.choice([1, 2, 5, 17])))
    monkeypatch.setenv("EARL_PLAN_PATH", "general")
    pg = ed.plan(src, dst, lens_dev, fields)
    monkeypatch.delenv("EARL_PLAN_PATH")
    pf = ed.plan(src, dst, lens_dev, fields)
    assert pf.hash() == pg.hash()
    if n <= 5000:
        assert pf.export() == O.route(src, dst, lens, world)
    dst_ranks = range(dst["rank0"], dst["rank0"] + dst["dp"] * dst["sp"] * dst["tp"])
    for r in dst_ranks:
        cu_f, ids_f, ts_f = ed.meta(pf, r)
        cu_g, ids_g, ts_g = ed.meta(pg, r)
        assert cu_f.cpu().tolist() == cu_g.cpu().tolist()
        assert ids_f.cpu().tolist() == ids_g.cpu().tolist()
        assert ts_f.cpu().tolist() == ts_g.cpu().tolist()
    pf.destroy()
    pg.destroy()
