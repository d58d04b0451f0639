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


def _digests(arrays, workers=16):
    """BLAKE2b-256 of each uint8 array (threads: hashlib releases the GIL on large buffers)."""
    import hashlib
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(workers) as ex:
        return list(ex.map(lambda a: hashlib.blake2b(memoryview(a), digest_size=32).hexdigest(),
                           arrays))


def _host_bytes_available():
    try:
        import psutil
        return psutil.virtual_memory().available
    except Exception:
        return None


@pytest.mark.parametrize("config,fields_name,ram_factor,n_seqs", [
    ("c3", "scalar6-fp32+hidden2560", 9, 512), ("c4", "scalar6-fp32+hidden8192", 3.5, 512),
    ("c2-lpt", "scalar6-fp32+hidden2560", 4, 512),
    ("c5-lt", "scalar6-fp32", 4, 39250)])  # the sweep's 256 MiB/rank long-tail point: misaligned
def test_bench_workload_full_digest_parity(config, fields_name, ram_factor, n_seqs):
    """SURVEY.md §8(c) GPU parity above 1 GB: the WHOLE bench batch (every byte of every field on
    every destination rank, TP replicas included) as BLAKE2b-256 digests per (rank, field), the
    GPU's fused exec (replan + exec, bench.py's launch) against the oracle's dispatch of the
    same source bytes.  c3 also checks the staged path (pack + unpack) the same way."""
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
    lens, src, dst, fields, _ = bench.workload(config, R, fields_name, n_seqs=n_seqs)
    lens = [int(x) for x in lens]
    F = len(fields)
    payload = sum(lens) * W.bytes_per_token(fields)
    avail = _host_bytes_available()
    if avail is not None and avail < ram_factor * payload:
        pytest.skip(f"host RAM {avail / 2**30:.0f} GiB < {ram_factor} x {payload / 2**30:.1f} GiB "
                    f"needed by the oracle for the full batch")
    tok_r = W.rollout_token_counts(lens, src["counts"])
    send = [W.gen_field_device(fields[f], tok_r[r], 1000 + 16 * r + f, dev)
            for r in range(R) for f in range(F)]
    ed = EmulatedDispatch(R)
    lens_dev = torch.as_tensor(np.asarray(lens, dtype=np.int32)).to(dev)
    plan = ed.plan(src, dst, lens_dev, fields)
    recv = ed.flat(ed.alloc_recv(plan, fields))
    for x in recv:
        x.fill_(0xA5)
    plan.replan(lens_dev)
    plan.exec(send, recv)
    torch.cuda.synchronize()
    plan.sync()
    gpu_exec = _digests([x.cpu().numpy() for x in recv])
    gpu_staged = None
    if config == "c3":
        for x in recv:
            x.fill_(0x5A)
        stage = ed.alloc_stage(plan)
        plan.pack(send, stage)
        plan.unpack(stage, recv)
        torch.cuda.synchronize()
        plan.sync()
        del stage
        gpu_staged = _digests([x.cpu().numpy() for x in recv])
    del recv
    src_arrays = {r: [send[r * F + f].cpu().numpy() for f in range(F)] for r in range(R) if tok_r[r]}
    del send
    torch.cuda.empty_cache()
    want, _, _ = O.dispatch(src, dst, lens, src_arrays, fields, R)
    del src_arrays
    ref = []
    for d in range(R):
        for f in range(F):
            ref.append(want[d][f] if d in want else np.zeros(0, np.uint8))
    ref = _digests(ref)
    del want
    for k, (g, w) in enumerate(zip(gpu_exec, ref)):
        assert g == w, (config, "exec", "rank", k // F, "field", k % F)
    if gpu_staged is not None:
        for k, (g, w) in enumerate(zip(gpu_staged, ref)):
            assert g == w, (config, "staged", "rank", k // F, "field", k % F)
    plan.destroy()


def test_midsize_tp4_hidden_element_by_element():
    """The bench's own copy-engine shape at scale, compared byte for byte: ~0.5 GB of
    scalar6 + hidden2560 (>= 90% of the bytes in 16-B-multiple fields, so the launch takes the
    congruent-heavy copy_kernel<2, 2, 16384> shape, 888 warps with ~8 dynamic work units each:
    unit claims, ring wrap-around and 4-replica TMA stores), DP8 -> DP2 x TP4, every byte of
    every replica against the oracle, with guard bands; fused exec and pack + unpack."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2510_05943_b200 import build
    from paper_2510_05943_b200 import workloads as W
    from tests.helpers import run_gpu_case
    build.build()
    lens = [int(x) for x in W.c2_lengths(3)[:48]]
    fields = W.field_set("scalar6-fp32+hidden2560")
    assert sum(lens) * W.bytes_per_token(fields) >= 200e6
    src, dst = W.config_layouts("c3", 8, len(lens))
    for mode in ("exec", "stage"):
        run_gpu_case(src, dst, lens, fields, 8, mode=mode, seed=5, check_plan=(mode == "exec"))
