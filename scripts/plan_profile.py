"""Planner cost at mid-size N: event-timed replan alone, exec alone and
replan + exec (steady state: one plan object re-planned every batch, nothing allocated), for the
C5 sweep's 256 MiB/rank points (uniform and long-tail scalar6, DP8 -> DP8 round-robin) and the
bench configs.  EARL_PLAN_TRACE=1 adds the in-kernel phase times on stderr.
Prints one JSON line per case."""
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
from paper_2510_05943_b200.earl import PtrArray  # noqa: E402

HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] * 1e9 \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6.65e12
R = 8
MiB = 1 << 20


def cases():
    f6 = W.field_set("scalar6-fp32")
    lt_mean = float(W.lognormal_lengths(100000, 2048, 0.75, 64, 8192, 0).mean())
    for kind, mib in (("uniform", 256), ("longtail", 256), ("longtail", 64), ("longtail", 1024)):
        n = int(round(mib * MiB * R / (21 * (4096 if kind == "uniform" else lt_mean))))
        lens = np.full(n, 4096) if kind == "uniform" else W.lognormal_lengths(n, 2048, 0.75, 64, 8192, 0)
        src = W.rollout_layout(n, R)
        dst = W.layout(dp=R, assign="explicit", group_of_seq=np.arange(n, dtype=np.int32) % R)
        yield f"c5-{kind}-{mib}MiB", lens, src, dst, f6
    for cfg in ("c3", "c2-lpt", "c4"):
        lens = W.c4_lengths(0) if cfg == "c4" else W.c2_lengths(0)
        src, dst = W.config_layouts(cfg, R, len(lens))
        yield f"{cfg}-scalar6", lens, src, dst, f6


def main():
    dev = torch.device("cuda", 0)
    flush = torch.empty(512 * MiB, dtype=torch.uint8, device=dev)
    ed = EmulatedDispatch(R)
    reps = int(os.environ.get("REPS", "20"))
    for name, lens, src, dst, fields in cases():
        F = len(fields)
        lens_dev = torch.as_tensor(np.asarray(lens, dtype=np.int32)).to(dev)
        tok = W.rollout_token_counts(lens, src["counts"])
        send = [W.gen_field_device(fields[f], tok[r], 1000 + 16 * r + f, dev)
                for r in range(R) for f in range(F)]
        plan = ed.plan(src, dst, lens_dev, fields)
        st = plan.stats()
        recv = PtrArray(ed.flat(ed.alloc_recv(plan, fields)))
        send = PtrArray(send)
        alg = sum(st["read_bytes"]) + st["total"]
        for _ in range(3):
            plan.replan(lens_dev)
            plan.exec(send, recv)
        torch.cuda.synchronize()
        tp, te, tt = [], [], []
        for _ in range(reps):
            flush.zero_()
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record()
            plan.replan(lens_dev)
            e[1].record()
            plan.exec(send, recv)
            e[2].record()
            torch.cuda.synchronize()
            tp.append(e[0].elapsed_time(e[1]))
            te.append(e[1].elapsed_time(e[2]))
            tt.append(e[0].elapsed_time(e[2]))
        m = statistics.median
        print(json.dumps({"case": name, "n_seqs": len(lens), "records": st["records"],
                          "alg_bytes": int(alg), "replan_ms": m(tp), "exec_ms": m(te),
                          "plan_exec_ms": m(tt), "exec_frac": alg / (m(te) * 1e-3) / HBM,
                          "plan_exec_frac": alg / (m(tt) * 1e-3) / HBM}), flush=True)
        plan.destroy()
        del send, recv
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
