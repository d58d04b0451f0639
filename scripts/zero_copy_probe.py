"""Probe: earl_dispatch_exec reading HOST-pinned (UVA-mapped) source buffers directly (the copy
kernel's TMA loads cross PCIe; no separate H2D), against H2D copies + exec from HBM.  Same c3 +
hidden2560 workload as bench.py; bytes compared against the device-source exec."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2510_05943_b200 import workloads as W  # noqa: E402
from paper_2510_05943_b200.dispatch import EmulatedDispatch  # noqa: E402

dev = torch.device("cuda", 0)
R = 8
lens, src, dst, fields, desc = bench.workload("c3", R, sys.argv[1] if len(sys.argv) > 1 else "scalar6-fp32+hidden2560")
F = len(fields)
ed = EmulatedDispatch(R)
stream = torch.cuda.current_stream()
lens_dev = torch.as_tensor(lens.astype(np.int32)).to(dev)
tok_r = W.rollout_token_counts(lens, src["counts"])
send = [W.gen_field_device(fields[f], tok_r[r], 1000 + 16 * r + f, dev) for r in range(R) for f in range(F)]
host = [torch.empty(t.numel(), dtype=torch.uint8, pin_memory=True) for t in send]
for h, d in zip(host, send):
    h.copy_(d)
plan = ed.plan(src, dst, lens_dev, fields, stream)
st = plan.stats()
payload = st["total_tokens"] * st["bytes_per_token"]
recv_a = ed.flat(ed.alloc_recv(plan, fields))
recv_b = ed.flat(ed.alloc_recv(plan, fields))
plan.exec(send, recv_a, stream)
torch.cuda.synchronize()
plan.exec(host, recv_b, stream)
torch.cuda.synchronize()
plan.sync()
same = all(torch.equal(a, b) for a, b in zip(recv_a, recv_b))
print("zero-copy bytes equal:", same, flush=True)


def timed(fn, n=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(n):
        fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


def h2d_exec():
    for h, d in zip(host, send):
        d.copy_(h, non_blocking=True)
    plan.replan(lens_dev, stream)
    plan.exec(send, recv_a, stream)


def zero_copy():
    plan.replan(lens_dev, stream)
    plan.exec(host, recv_b, stream)


def h2d_only():
    for h, d in zip(host, send):
        d.copy_(h, non_blocking=True)


for name, fn in (("h2d only", h2d_only), ("h2d + replan + exec", h2d_exec), ("zero-copy replan + exec", zero_copy)):
    ms = timed(fn)
    print(f"{name:28s} {ms:8.2f} ms  {payload / ms / 1e6:6.1f} GB/s", flush=True)
