"""Parity at BASELINE.json's full size, in the launch configuration bench.py times.

The bench workload (config 3 on configs[1]'s 512-episode batch, scalar6-fp32 + hidden2560,
6.78 GB, 8-rank emulation DP8 -> DP2 x TP4, device-drawn payloads with bench.py's seeds) is
planned, re-planned and dispatched exactly as the timed loop does.  The oracle computes, one by
one, where sampled sequences live on the source and on every destination replica; their bytes
must be equal.  For the whole batch, a property that holds at any size: per field and per TP
replica, the destination bytes sum to the source bytes (every token exactly once per replica).
"""
import numpy as np
import pytest

from oracle import earl_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("config,fields_name", [("c3", "scalar6-fp32+hidden2560"),
                                                ("c4", "scalar6-fp32+hidden8192")])
def test_bench_workload_sampled_parity(config, fields_name):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import bench
    from paper_2510_05943_b200 import build
    from paper_2510_05943_b200 import workloads as W
    from paper_2510_05943_b200.dispatch import EmulatedDispatch
    build.build()
    dev = torch.device("cuda", 0)
    R = 8
    lens, src, dst, fields, _ = bench.workload(config, R, fields_name)
    lens = [int(x) for x in lens]
    F = len(fields)
    Bf = [b * e for (_, b, e, _) in fields]
    tok_r = W.rollout_token_counts(lens, src["counts"])
    send = [W.gen_field_device(fields[f], tok_r[r], 1000 + 16 * r + f, dev)
            for r in range(R) for f in range(F)]
    ed = EmulatedDispatch(R)
    lens_dev = torch.as_tensor(np.asarray(lens, dtype=np.int32)).to(dev)
    plan = ed.plan(src, dst, lens_dev, fields)
    recv = ed.flat(ed.alloc_recv(plan, fields))
    for x in recv:
        x.fill_(0xA5)
    plan.replan(lens_dev)  # the timed loop's step: replan + exec
    plan.exec(send, recv)
    torch.cuda.synchronize()
    plan.sync()

    hs = O.holdings(src, lens, O.assign_groups(src, lens))
    hd = O.holdings(dst, lens, O.assign_groups(dst, lens))
    where_src = {}
    for r, h in hs.items():
        for (i, c, lo, hi) in h["chunks"]:
            where_src[i] = (r, h["local_off"][(i, c)])
    rng = np.random.default_rng(11)
    N = len(lens)
    sample = {0, 1, N - 1, int(np.argmax(lens)), int(np.argmin(lens))}
    sample |= set(rng.choice(N, 20, replace=False).tolist())
    checked = 0
    for d, h in hd.items():
        for (i, c, lo, hi) in h["chunks"]:
            if i not in sample or hi == lo:
                continue
            s, so = where_src[i]
            do = h["local_off"][(i, c)]
            for f in range(F):
                b = Bf[f]
                want = send[s * F + f][(so + lo) * b:(so + hi) * b].cpu().numpy()
                got = recv[d * F + f][do * b:(do + hi - lo) * b].cpu().numpy()
                assert np.array_equal(got, want), (config, "seq", i, "dst rank", d, "field", f)
            checked += 1
    assert checked >= len(sample) * dst["tp"] * dst["sp"] - 5

    # whole batch: byte sums per field and per TP replica equal the source's
    for f in range(F):
        src_sum = sum(int(send[r * F + f].to(torch.int64).sum()) for r in range(R) if tok_r[r])
        for t in range(dst["tp"]):
            dst_sum = sum(int(recv[d * F + f].to(torch.int64).sum())
                          for d in hd if O.coords_of(dst, d)[2] == t and recv[d * F + f].numel())
            assert dst_sum == src_sum, (config, "field", f, "replica", t)
    plan.destroy()
