"""Shared test helpers: random layouts and the GPU-vs-oracle case runner."""
import random

import numpy as np

from oracle import earl_oracle as O
from paper_2510_05943_b200 import workloads as W


def random_layout(rng: random.Random, world: int, n: int, allow_lpt=True):
    while True:
        dp = rng.randint(1, world)
        sp = rng.randint(1, max(1, world // dp))
        tp = rng.randint(1, max(1, world // (dp * sp)))
        if dp * sp * tp <= world:
            break
    rank0 = rng.randint(0, world - dp * sp * tp)
    choices = ["given_counts", "contig", "explicit"] + (["lpt"] if allow_lpt else [])
    a = rng.choice(choices)
    counts = gos = None
    if a == "given_counts":
        cuts = sorted(rng.randint(0, n) for _ in range(dp - 1))
        counts = [b - a_ for a_, b in zip([0] + cuts, cuts + [n])]
    if a == "explicit":
        gos = [rng.randrange(dp) for _ in range(n)]
    return W.layout(rank0=rank0, dp=dp, sp=sp, tp=tp, assign=a, counts=counts, group_of_seq=gos)


def run_gpu_case(src, dst, lens, fields, world, mode="exec", seed=0, check_plan=True,
                 guard=256, ed=None, host_src=False):
    """Dispatch on the GPU (emulated comm) and compare byte for byte with the oracle.

    mode: "exec" (fused direct), "exec_src" (fused, one launch per source rank) or "stage"
    (pack + unpack).  host_src: the source arrays are
    pinned HOST memory read by the kernels over PCIe (zero-copy).  Returns the plan stats."""
    import torch
    from paper_2510_05943_b200.dispatch import EmulatedDispatch

    lens = [int(x) for x in lens]
    T = sum(lens)
    glob = W.gen_global_fields(fields, T, seed_base=seed * 31 + 7, random_bits=True)
    gs = O.assign_groups(src, lens)
    src_arrays = O.rank_arrays_from_global(src, lens, gs, glob, fields)
    want, meta, segs = O.dispatch(src, dst, lens, src_arrays, fields, world)

    ed = ed or EmulatedDispatch(world)
    plan = ed.plan(src, dst, lens, fields)
    if check_plan:
        got = plan.export()
        assert got == segs, _first_diff(got, segs)
    st = plan.stats()
    Bf = O.field_bytes(fields)
    dev = ed.device
    send = []
    for r in range(world):
        for f in range(len(fields)):
            if r in src_arrays and src_arrays[r][f].size:
                t = torch.from_numpy(src_arrays[r][f])
                send.append(t.pin_memory() if host_src else t.to(dev))
            else:
                send.append(None)
    bufs, recv = [], []
    for r in range(world):
        n_tok = int(st["n_local_tokens"][r])
        if r in want:
            assert n_tok == O.holdings(dst, lens, O.assign_groups(dst, lens))[r]["n_tokens"]
        for f in range(len(fields)):
            n = n_tok * Bf[f]
            buf = torch.full((n + 2 * guard,), 0xA5, dtype=torch.uint8, device=dev)
            bufs.append((buf, n))
            recv.append(buf[guard:guard + n] if n else None)
    if mode == "exec":
        plan.exec(send, recv)
    elif mode == "exec_src":  # one launch per source rank, in a seeded random order
        order = list(range(world))
        random.Random(seed).shuffle(order)
        for r in order:
            plan.exec_src(r, send, recv)
    else:
        stage = ed.alloc_stage(plan)
        for s_ in stage:
            s_.fill_(0x5A)
        plan.pack(send, stage)
        plan.unpack(stage, recv)
    torch.cuda.synchronize()
    plan.sync()
    for r in range(world):
        for f in range(len(fields)):
            buf, n = bufs[r * len(fields) + f]
            host = buf.cpu().numpy()
            assert np.all(host[:guard] == 0xA5) and np.all(host[guard + n:] == 0xA5), \
                f"write outside rank {r} field {f}"
            if r in want:
                assert np.array_equal(host[guard:guard + n], want[r][f]), f"rank {r} field {f} differs"
            else:
                assert n == 0
    # destination metadata
    for r, m in meta.items():
        cu, ids, ts = ed.meta(plan, r)
        assert cu.cpu().tolist() == m["cu_seqlens"]
        assert ids.cpu().tolist() == m["seq_ids"]
        assert ts.cpu().tolist() == m["tok_start"]
    ostats = O.stats(segs, fields, world)
    assert [row[:world] for row in st["C"]] == ostats["C"]
    assert st["moved"] == ostats["moved"] and st["total"] == ostats["total"]
    assert st["segments"] == len(segs)
    plan.destroy()
    return st


def _first_diff(a, b):
    for k, (x, y) in enumerate(zip(a, b)):
        if x != y:
            return f"segment {k}: gpu {x} vs oracle {y}"
    return f"lengths {len(a)} vs {len(b)}"
