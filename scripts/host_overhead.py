"""Host-side cost of one call through the binding and the C ABI (ctypes marshalling + argument
checks + launch), measured while the GPU is held busy so the calls only enqueue: replan, exec,
and the a1 gather of the emulated comm, on the bench's c3 layouts.  Also the c0 floor step
(512 empty sequences) eager against a replayed CUDA graph.  One JSON line."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_05943_b200 import workloads as W  # noqa: E402
from paper_2510_05943_b200.dispatch import EmulatedDispatch, rank_counts  # noqa: E402


def host_us(fn, n=200):
    # one untimed call first: the first launch of a kernel loads its module lazily, which waits
    # for the device (here: the whole sleep), and would read as ~250 us per call
    fn()
    torch.cuda.synchronize()
    torch.cuda._sleep(2_000_000_000 // 1000 * 50)  # ~50 ms of GPU time ahead of the calls
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return (t1 - t0) / n * 1e6


def main():
    dev = torch.device("cuda", 0)
    R = 8
    lens = W.c2_lengths(0)
    src, dst = W.config_layouts("c3", R, len(lens))
    fields = W.field_set("scalar6-fp32")
    ed = EmulatedDispatch(R)
    lens_dev = torch.as_tensor(np.asarray(lens, dtype=np.int32)).to(dev)
    plan = ed.plan(src, dst, lens_dev, fields)
    recv = ed.flat(ed.alloc_recv(plan, fields))
    tok = W.rollout_token_counts(lens, src["counts"])
    send = [W.gen_field_device(fields[f], tok[r], 7 + f, dev) for r in range(R) for f in range(len(fields))]
    counts = rank_counts(src, R)
    edges = np.concatenate([[0], np.cumsum(counts)]).astype(int)
    loc = [torch.as_tensor(np.asarray(lens[edges[r]:edges[r + 1]], dtype=np.int32)).to(dev) for r in range(R)]
    from paper_2510_05943_b200.earl import PtrArray
    ps, pr = PtrArray(send), PtrArray(recv)
    out = {"note": "host us per call while the GPU is busy (includes any launch-queue back-pressure)",
           "replan_us": host_us(lambda: plan.replan(lens_dev)),
           "exec_us": host_us(lambda: plan.exec(send, recv)),
           "exec_prebuilt_ptrs_us": host_us(lambda: plan.exec(ps, pr)),
           "gather_us": host_us(lambda: ed.allgather_lens(loc, counts, out=lens_dev))}
    # the c0 floor: eager step against a replayed graph (device time, CUDA events)
    z = torch.zeros(512, dtype=torch.int32, device=dev)
    p0 = ed.plan(src, dst, z, fields)
    r0 = ed.flat(ed.alloc_recv(p0, fields))

    ps0, pr0 = PtrArray(send), PtrArray(r0)

    def step(s=None):
        p0.replan(z, s)
        p0.exec(ps0, pr0, s)

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(100):
        step()
    b.record()
    torch.cuda.synchronize()
    out["c0_eager_us"] = a.elapsed_time(b) / 100 * 1e3
    gs = torch.cuda.Stream()
    gs.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=gs):
        step(gs)
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    a.record()
    for _ in range(100):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    out["c0_graph_us"] = a.elapsed_time(b) / 100 * 1e3
    print(json.dumps(out))


if __name__ == "__main__":
    main()
