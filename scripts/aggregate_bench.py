"""NEXT-2 measurement: earl_returns + earl_advantages on the source ranks (8-rank emulation),
HBM-bound.  Algorithmic bytes per token: returns read r (4) + m (1), write G (4); advantages
read G (4) + m (1), write A (4): 18 B/token."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_05943_b200 import workloads as W  # noqa: E402
from paper_2510_05943_b200.dispatch import EmulatedDispatch  # noqa: E402

import argparse  # noqa: E402
ap = argparse.ArgumentParser()
ap.add_argument("--only", default="", help="substring of the workload name")
ap.add_argument("--iters", type=int, default=13)
args = ap.parse_args()
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] * 1e9
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for name, lens in (("C2 batch (512 x <=8K)", W.c2_lengths(0)),
                   ("C4 batch (256 x 4K-32K)", W.c4_lengths(0)),
                   ("C5-lt 131K episodes", W.lognormal_lengths(131072, 2048, 0.75, 64, 8192, 0))):
    if args.only not in name:
        continue
    n = len(lens)
    src = W.rollout_layout(n, 8)
    ed = EmulatedDispatch(8)
    plan = ed.plan(src, W.layout(dp=2, tp=4, assign="contig"), lens, W.field_set("tiny3"))
    plan.sync()  # the host learns the batch's size (as any caller sizing its buffers does)
    tok = W.rollout_token_counts(lens, src["counts"])
    r = [torch.randn(max(t, 1), device="cuda") for t in tok]
    m = [(torch.rand(max(t, 1), device="cuda") < 0.8).to(torch.uint8) for t in tok]
    G = [torch.empty(max(t, 1), device="cuda") for t in tok]
    A = [torch.empty(max(t, 1), device="cuda") for t in tok]
    part = torch.zeros(3, dtype=torch.float64, device="cuda")
    ts = []
    for k in range(args.iters):
        flush.zero_()
        part.zero_()
        a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a.record()
        plan.returns(0.99, r, m, G, part)
        b.record()
        plan.advantages(part, 1e-8, G, m, A)
        c.record()
        torch.cuda.synchronize()
        if k >= 3:
            ts.append((a.elapsed_time(b), b.elapsed_time(c)))
    T = sum(tok)
    tr = float(np.median([x[0] for x in ts]))
    ta = float(np.median([x[1] for x in ts]))
    print(json.dumps({"workload": name, "tokens": T, "returns_ms": tr, "advantages_ms": ta,
                      "returns_hbm_frac": 9 * T / (tr * 1e-3) / peak,
                      "advantages_hbm_frac": 9 * T / (ta * 1e-3) / peak}))
