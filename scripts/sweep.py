"""C5 bandwidth sweep (BASELINE.json configs[4]) on one B200, 8-rank emulation.

For payload P per rank in 1 MiB .. 4 GiB, uniform (L = 4096) and long-tail (C2 distribution)
lengths, scalar6-fp32 fields (series A) and +hidden2560 (series B, P >= 64 MiB):
  * a2a  : earl_plan_replan + earl_dispatch_exec, DP8 -> DP8 EXPLICIT round-robin
           (uniform all-to-allv), i.e. the decentralized dispatch;
  * cent : the centralized gather-and-dispatch baseline (reading c13): DP8 ->
           DP1 on rank 0, then DP1 -> DP8, two replans + two execs.
Times are CUDA-event medians with an L2 flush before every timed repetition.  Beside the
measured (HBM-bound, one GPU) times it reports the NVLink model of SURVEY.md §8(d):
t_a2a = max_r max(egress_r, ingress_r) / 770 GB/s, t_cent = (ingress_0 + egress_0) / 770 GB/s
(the controller's link serialises both phases).  Writes profiles/<tag>_sweep.json.
"""
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

NVL = 770e9
HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] * 1e9 \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6.65e12
R = 8
MiB = 1 << 20


def lengths(kind, n):
    if kind == "uniform":
        return np.full(n, 4096, dtype=np.int64)
    return W.lognormal_lengths(n, 2048, 0.75, 64, 8192, 0)


def n_for(kind, fields, per_rank):
    B = W.bytes_per_token(fields)
    mean = 4096 if kind == "uniform" else float(W.lognormal_lengths(100000, 2048, 0.75, 64, 8192, 0).mean())
    return max(R, int(round(per_rank * R / (B * mean))))


def timed(fn, reps, flush):
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


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
    dev = torch.device("cuda", 0)
    flush = torch.empty(512 * MiB, dtype=torch.uint8, device=dev)
    ed = EmulatedDispatch(R)
    rows = []
    only = os.environ.get("SWEEP_ONLY", "")  # e.g. "B:longtail:1024" (re-measure one point)
    for series, fname in (("A", "scalar6-fp32"), ("B", "scalar6-fp32+hidden2560")):
        fields = W.field_set(fname)
        F = len(fields)
        for kind in ("uniform", "longtail"):
            for p_mib in (1, 4, 16, 64, 256, 1024, 4096):
                if series == "B" and p_mib < 64:
                    continue
                if only and only != f"{series}:{kind}:{p_mib}":
                    continue
                n = n_for(kind, fields, p_mib * MiB)
                lens = lengths(kind, n)
                src = W.rollout_layout(n, R)
                dst = W.layout(dp=R, assign="explicit", group_of_seq=np.arange(n, dtype=np.int32) % R)
                mid = W.layout(dp=1, assign="given_counts", counts=[n])
                tok = W.rollout_token_counts(lens, src["counts"])
                send = [W.gen_field_device(fields[f], tok[r], 1000 + 16 * r + f, dev)
                        for r in range(R) for f in range(F)]
                lens_dev = torch.as_tensor(lens.astype(np.int32)).to(dev)
                p_a = ed.plan(src, dst, lens_dev, fields)
                p_1 = ed.plan(src, mid, lens_dev, fields)
                p_2 = ed.plan(mid, dst, lens_dev, fields)
                st_a, st_1, st_2 = p_a.stats(), p_1.stats(), p_2.stats()
                recv = ed.flat(ed.alloc_recv(p_a, fields))
                midb = ed.flat(ed.alloc_recv(p_1, fields))
                recv2 = ed.flat(ed.alloc_recv(p_2, fields))
                # pointer arrays marshalled once: small sizes are otherwise host-bound
                send, recv, midb, recv2 = (PtrArray(x) for x in (send, recv, midb, recv2))

                # steady state (the timed region allocates nothing): the plan
                # objects are made once and every repetition re-plans the batch on the device
                # (earl_plan_replan) before dispatching it
                def a2a():
                    p_a.replan(lens_dev)
                    p_a.exec(send, recv)

                def cent():
                    p_1.replan(lens_dev)
                    p_1.exec(send, midb)
                    p_2.replan(lens_dev)
                    p_2.exec(midb, recv2)

                for _ in range(2):
                    a2a(); cent()
                torch.cuda.synchronize()
                reps = 10 if p_mib <= 1024 else 4
                t_a = timed(a2a, reps, flush)
                t_c = timed(cent, reps, flush)
                payload = st_a["total_tokens"] * st_a["bytes_per_token"]
                hbm_a = sum(st_a["read_bytes"]) + st_a["total"]
                nvl_a = max(max(st_a["egress"]), max(st_a["ingress"])) / NVL * 1e3
                nvl_c = (st_1["ingress"][0] + st_2["egress"][0]) / NVL * 1e3
                row = {"series": series, "fields": fname, "lengths": kind, "per_rank_MiB": p_mib,
                       "n_seqs": int(n), "payload_bytes": int(payload),
                       "a2a_ms": t_a, "cent_ms": t_c, "measured_ratio": t_c / t_a,
                       "a2a_GBps": payload / t_a / 1e6, "a2a_hbm_frac": hbm_a / (t_a * 1e-3) / HBM,
                       "nvlink_model_a2a_ms": nvl_a, "nvlink_model_cent_ms": nvl_c,
                       "nvlink_model_ratio": nvl_c / nvl_a if nvl_a else None,
                       "moved_a2a": st_a["moved"], "moved_cent": st_1["moved"] + st_2["moved"]}
                rows.append(row)
                print(json.dumps(row), flush=True)
                for q in (p_a, p_1, p_2):
                    q.destroy()
                del send, recv, midb, recv2
                torch.cuda.empty_cache()
    out = os.path.join(ROOT, "gpurun_out", f"{tag}_sweep.json")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    json.dump({"about": __doc__, "hbm_peak_Bps": HBM, "nvlink_Bps": NVL, "rows": rows}, open(out, "w"), indent=1)
    write_md(rows, tag, out[:-5] + ".md")


def write_md(rows, tag, path):
    head = [
        f"# C5 bandwidth sweep, {tag} (1 B200, 8-rank emulation; scripts/sweep.py)", "",
        "a2a = replan + fused exec (DP8 -> DP8 round-robin all-to-allv; the plan object made once, nothing "
        "allocated in the timed region); cent = centralized gather-and-dispatch via rank 0 (two replans + two execs).",
        "Measured times are CUDA-event medians with an L2 flush before each repetition. On one GPU every byte "
        "moves through HBM, so the",
        "measured centralized/a2a ratio is ~2 (two passes). The NVLink columns are the SURVEY.md §8(d) model "
        "for a real 8-GPU box",
        "(bottleneck link bytes / 770 GB/s): the controller serialises both phases, ratio = 2W = 16 for "
        "uniform payloads.", "",
        "| series | lengths | MiB/rank | N | a2a ms | a2a GB/s | HBM frac | cent ms | measured ratio | "
        "NVLink model a2a ms | NVLink model cent ms | model ratio |",
        "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    lines = []
    for r in rows:
        lines.append(
            f"| {r['series']} ({r['fields']}) | {'uniform' if r['lengths'] == 'uniform' else 'longtail'} | "
            f"{r['per_rank_MiB']} | {r['n_seqs']} | {r['a2a_ms']:.3f} | {r['a2a_GBps']:.0f} | "
            f"{r['a2a_hbm_frac']:.3f} | {r['cent_ms']:.3f} | {r['measured_ratio']:.2f} | "
            f"{r['nvlink_model_a2a_ms']:.3f} | {r['nvlink_model_cent_ms']:.3f} | "
            f"{(r['nvlink_model_ratio'] or 0):.1f} |")
    open(path, "w").write("\n".join(head + lines) + "\n")


if __name__ == "__main__":
    main()
