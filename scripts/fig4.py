"""The paper's dispatch experiment (Fig. 4) replayed on one B200 (8-rank
emulation): per worker the log-probs of 1500 responses padded to the context length L, fp32
(46.875 / 93.75 / 187.5 MiB per worker at L = 8K / 16K / 32K: the paper's "46, 93 and 187 MB";
the 1500 x L x 4 B factorisation is SURVEY.md §6's reading).  Rollout/reference DP8 ->
training DP2 x TP4 (CONTIG):
  * EARL   : one decentralized dispatch (plan + fused exec), PAPER.md:195-196;
  * central: gather every worker's tensor on the controller (rank 0) and scatter it to the
             trainers (reading c13): two dispatches.
Measured on one GPU both are HBM-bound (every byte moves through one HBM); the NVLink column is
the 8-GPU model of SURVEY.md §8(d): max_r max(egress_r, ingress_r) / 770 GB/s for EARL, the
controller's ingress + egress / 770 GB/s for the centralized path.  The paper's own ratios
(9.7x at 8K, 11.2x at 32K) were measured over TCP between 16 nodes: context, not a target."""
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_05943_b200 import workloads as W  # noqa: E402
from paper_2510_05943_b200.dispatch import EmulatedDispatch  # noqa: E402

R, NVL = 8, 770e9
dev = torch.device("cuda", 0)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
fields = [("old_logprobs", 4, 1, "logprob")]


def timed(fn, reps=10):
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


ed = EmulatedDispatch(R)
for L in W.FIG4_CONTEXTS:
    lens = W.fig4_lengths(L, R)
    n = len(lens)
    src = W.rollout_layout(n, R)
    dst = W.layout(dp=2, tp=4, assign="contig")
    mid = W.layout(dp=1, assign="given_counts", counts=[n])
    tok = W.rollout_token_counts(lens, src["counts"])
    send = [W.gen_field_device(fields[0], tok[r], 1000 + 16 * r, dev) for r in range(R)]
    ld = torch.as_tensor(lens.astype(np.int32)).to(dev)
    pa, p1, p2 = ed.plan(src, dst, ld, fields), ed.plan(src, mid, ld, fields), ed.plan(mid, dst, ld, fields)
    sa, s1, s2 = pa.stats(), p1.stats(), p2.stats()
    recv = ed.flat(ed.alloc_recv(pa, fields))
    midb = ed.flat(ed.alloc_recv(p1, fields))
    recv2 = ed.flat(ed.alloc_recv(p2, fields))

    def earl():
        pa.replan(ld)
        pa.exec(send, recv)

    def central():
        p1.replan(ld)
        p1.exec(send, midb)
        p2.replan(ld)
        p2.exec(midb, recv2)

    for _ in range(2):
        earl(); central()
    torch.cuda.synchronize()
    same = all(torch.equal(x, y) for x, y in zip(recv, recv2))
    t_e, t_c = timed(earl), timed(central)
    worker_mib = tok[0] * 4 / (1 << 20)
    nvl_e = max(max(sa["egress"]), max(sa["ingress"])) / NVL * 1e3
    nvl_c = (s1["ingress"][0] + s2["egress"][0]) / NVL * 1e3
    print(json.dumps({"context": L, "per_worker_MiB": worker_mib, "earl_ms": t_e, "central_ms": t_c,
                      "measured_ratio_1gpu": t_c / t_e, "nvlink_model_earl_ms": nvl_e,
                      "nvlink_model_central_ms": nvl_c, "nvlink_model_ratio": nvl_c / nvl_e,
                      "same_bytes": same, "moved_earl": sa["moved"],
                      "moved_central": s1["moved"] + s2["moved"]}), flush=True)
    for q in (pa, p1, p2):
        q.destroy()
    del send, recv, midb, recv2
    torch.cuda.empty_cache()
