"""GPU: step a1 on the device (earl_allgather_lengths) chained into the planner and the fused
exec -- directly and as one captured CUDA graph -- and the plan's cross-stream ordering
(every launch on a plan waits for the previous one; earl_plan_sync / destroy cover them all).

The multi-process form of a1 (stores into peer windows + epoch flags) runs in
tests/test_multiprocess.py (mp_worker.gpu_main gathers every rank's local lengths before
planning)."""
import numpy as np
import pytest

from oracle import earl_oracle as O
from paper_2510_05943_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2510_05943_b200 import build
    build.build()


def _rank_major(lens, counts):
    edges = np.concatenate([[0], np.cumsum(counts)]).astype(int)
    return [list(lens[edges[r]:edges[r + 1]]) for r in range(len(counts))]


@pytest.mark.parametrize("seed", range(6))
def test_emulated_gather_is_rank_major_concatenation(seed):
    import torch
    from paper_2510_05943_b200.dispatch import EmulatedDispatch
    rng = np.random.default_rng(seed)
    world = int(rng.integers(1, 9))
    counts = [int(c) for c in rng.integers(0, 700, size=world)]
    if seed == 0:
        counts = [0] * world          # nothing at all
    elif seed == 1:
        counts[0] = 0                 # a rank with no sequences of its own
    lens = rng.integers(0, 9000, size=sum(counts)).astype(np.int32)
    ed = EmulatedDispatch(world)
    loc = [torch.as_tensor(np.asarray(x, dtype=np.int32)).cuda() if len(x) else None
           for x in _rank_major(lens, counts)]
    got = ed.allgather_lens(loc, counts)
    torch.cuda.synchronize()
    assert got.cpu().numpy().tolist() == lens.tolist()


def test_gathered_lengths_plan_equals_oracle_plan():
    import torch
    from paper_2510_05943_b200.dispatch import EmulatedDispatch, rank_counts
    lens = W.c2_lengths(0)
    world = 8
    src, dst = W.config_layouts("c3", world, len(lens))
    counts = rank_counts(src, world)
    ed = EmulatedDispatch(world)
    loc = [torch.as_tensor(np.asarray(x, dtype=np.int32)).cuda() if len(x) else None
           for x in _rank_major(lens, counts)]
    glens = ed.allgather_lens(loc, counts)
    fields = W.field_set("tiny3")
    plan = ed.plan(src, dst, glens, fields)
    segs = O.route(src, dst, [int(x) for x in lens], world)
    assert plan.export() == segs
    plan.destroy()


def test_gather_replan_exec_as_one_graph():
    """a1 gather + replan + exec captured once; every replay dispatches a new batch whose
    lengths exist only as per-rank local vectors -- bit-exact against the oracle each time."""
    import torch
    from paper_2510_05943_b200.dispatch import EmulatedDispatch, rank_counts
    world, n = 8, 160
    fields = [("ids", 4, 1, "x"), ("m", 1, 1, "x"), ("h", 2, 24, "x")]
    Bf = O.field_bytes(fields)
    rng = np.random.default_rng(7)
    batches = [rng.integers(0, 500, size=n) for _ in range(4)]
    src = W.rollout_layout(n, world)
    dst = W.layout(dp=2, tp=4, assign="contig")
    counts = rank_counts(src, world)
    cap = max(int(b.sum()) for b in batches)
    ed = EmulatedDispatch(world)
    dev = ed.device
    local = [torch.zeros(max(1, c), dtype=torch.int32, device=dev) for c in counts]
    glens = torch.zeros(n, dtype=torch.int32, device=dev)
    send = [torch.zeros(cap * b, dtype=torch.uint8, device=dev) for _ in range(world) for b in Bf]
    recv = [torch.zeros(cap * b, dtype=torch.uint8, device=dev) for _ in range(world) for b in Bf]

    def load(lens, seed):
        lens = [int(x) for x in lens]
        for r, x in enumerate(_rank_major(np.asarray(lens), counts)):
            if len(x):
                local[r][: len(x)].copy_(torch.as_tensor(np.asarray(x, dtype=np.int32)))
        glob = W.gen_global_fields(fields, sum(lens), seed_base=seed, random_bits=True)
        src_arrays = O.rank_arrays_from_global(src, lens, O.assign_groups(src, lens), glob, fields)
        want, meta, segs = O.dispatch(src, dst, lens, src_arrays, fields, world)
        for r in range(world):
            for f in range(len(fields)):
                a = src_arrays[r][f]
                if a.size:
                    send[r * len(fields) + f][: a.size].copy_(torch.from_numpy(a))
        return want, segs

    want, segs = load(batches[0], 3)
    ed.allgather_lens(local, counts, out=glens)
    plan = ed.plan(src, dst, glens, fields)
    plan.exec(send, recv)
    torch.cuda.synchronize()
    assert plan.export() == segs
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        ed.allgather_lens(local, counts, out=glens, stream=s)
        plan.replan(glens, stream=s)
        plan.exec(send, recv, stream=s)
    for k, lens in enumerate(batches[1:]):
        want, segs = load(lens, 40 + k)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        assert glens.cpu().numpy().tolist() == [int(x) for x in lens]
        assert plan.export() == segs
        for r, arrs in want.items():
            for f in range(len(fields)):
                got = recv[r * len(fields) + f][: arrs[f].size].cpu().numpy()
                assert np.array_equal(got, arrs[f]), (k, r, f)
    plan.destroy()


def test_plan_launches_ordered_across_streams():
    """plan on one stream, exec on another, exec_src on a third, destroy
    right away -- the launches run in issue order, plan.sync() waits for the last of them, and
    the plan's memory outlives the kernels that read it."""
    import torch
    from paper_2510_05943_b200.dispatch import EmulatedDispatch
    world = 8
    lens = [int(x) for x in W.c2_lengths(0)[:256]]
    fields = [("a", 4, 1, "x"), ("h", 2, 512, "x")]
    src, dst = W.config_layouts("c3", world, len(lens))
    glob = W.gen_global_fields(fields, sum(lens), seed_base=5, random_bits=True)
    src_arrays = O.rank_arrays_from_global(src, lens, O.assign_groups(src, lens), glob, fields)
    want, _, _ = O.dispatch(src, dst, lens, src_arrays, fields, world)
    ed = EmulatedDispatch(world)
    dev = ed.device
    send = [torch.from_numpy(src_arrays[r][f]).to(dev) if r in src_arrays else None
            for r in range(world) for f in range(len(fields))]
    s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    lens_dev = torch.as_tensor(np.asarray(lens, dtype=np.int32)).to(dev)
    torch.cuda.synchronize()
    with torch.cuda.stream(s1):
        plan = ed.plan(src, dst, lens_dev, fields, stream=s1)
    recv = ed.flat(ed.alloc_recv(plan, fields))
    for t in recv:
        t.fill_(0)
    torch.cuda.synchronize()
    for rep in range(3):
        with torch.cuda.stream(s1):
            plan.replan(lens_dev, stream=s1)
        plan.exec(send, recv, stream=s2)        # waits for the replan on s1
        for r in range(world):
            plan.exec_src(r, send, recv, stream=s3 if r % 2 else s2)
        plan.sync()                             # covers the launches on s2 and s3
        host = [t.cpu().numpy() for t in recv]  # read on the current stream, no device sync
        for r, arrs in want.items():
            for f in range(len(fields)):
                assert np.array_equal(host[r * len(fields) + f], arrs[f]), (rep, r, f)
    plan.exec(send, recv, stream=s3)
    plan.destroy()                              # freed after the exec on s3, stream-ordered
    torch.cuda.synchronize()
