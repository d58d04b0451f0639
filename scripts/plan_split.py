"""Plan vs exec split at the C5 sweep's 256 MiB/rank and 1 GiB/rank points (8-rank emulation),
plus the planner's phase trace (EARL_PLAN_TRACE=1 prints it)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2510_05943_b200 import workloads as W  # noqa: E402
from paper_2510_05943_b200.dispatch import EmulatedDispatch  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
for cfg, n in (("c5", 24966), ("c5-lt", 39250), ("c5", 99864), ("c5-lt", 157000)):
    lens, src, dst, fields, desc = bench.workload(cfg, 8, "scalar6-fp32", n)
    ed = EmulatedDispatch(8)
    ld = torch.as_tensor(lens.astype(np.int32)).to(dev)
    tok_r = W.rollout_token_counts(lens, src["counts"])
    F = len(fields)
    send = [W.gen_field_device(fields[f], tok_r[r], 1000 + 16 * r + f, dev) for r in range(8) for f in range(F)]
    plan = ed.plan(src, dst, ld, fields)
    recv = ed.flat(ed.alloc_recv(plan, fields))
    st = plan.stats()
    alg = sum(st["read_bytes"]) + st["total"]
    tp, te = [], []
    for k in range(8):
        flush.zero_()
        a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a.record()
        plan.replan(ld)
        b.record()
        plan.exec(send, recv)
        c.record()
        torch.cuda.synchronize()
        if k >= 2:
            tp.append(a.elapsed_time(b)); te.append(b.elapsed_time(c))
    tp, te = float(np.median(tp)), float(np.median(te))
    peak = bench.measured_peaks()[0]
    print(f"{cfg:6s} N={n:7d} plan {tp:.3f} ms  exec {te:.3f} ms  exec frac {alg / te / 1e6 / peak:.3f}  "
          f"plan+exec frac {alg / (tp + te) / 1e6 / peak:.3f}", flush=True)
    plan.destroy()
