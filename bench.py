#!/usr/bin/env python
"""bench.py -- EARL layout-aware dispatch on B200 (BASELINE.json metric: "dispatch GB/s per GPU &
ms/batch at 1/2/4/8 B200; % of NVLink/HBM roofline").

A step is one pass of the whole hot path over one batch: the global length
vector, the device planner (earl_dispatch_plan) and the dispatch itself (earl_dispatch_exec:
one fused pass that reads each source byte once and writes it at its final offset on every
destination replica).

  N = 1 : BASELINE.json configs[2] ("same batch exchanged rollout DP8 -> train DP2 x TP4") as an
          8-rank emulation on one B200 -- the batch of configs[1] (512 episodes, long tail <= 8192,
          6 per-token fields + a 4B-class hidden vector of width 2560), every emulated rank's
          bytes moved by one launch.  The staged pack/unpack path is timed beside it.
  N > 1 : one process per GPU (torchrun), DPn -> DP max(1,n/4) x TP min(4,n), the same batch
          (strong scaling), fused P2P stores over NVLink into symmetric windows.

  --impl reference : the CPU oracle (oracle/earl_oracle.py) on the host cores, bounded sample.

Prints one JSON line (rank 0).  Inputs are larger than L2 (6.3 GiB per batch), so no L2 flush.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "dispatch GB/s per GPU & ms/batch at 1/2/4/8 B200; % of NVLink/HBM roofline"
NVLINK_PEER_GBPS = 770.0   # B200_PROFILING.md: measured peer copy per direction (nominal 900)
NVLINK_NOMINAL_GBPS = 900.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c3", choices=["c3", "c4", "c2-lpt", "c5", "c5-lt", "c0"])
    ap.add_argument("--n-seqs", type=int, default=512, help="c5/c5-lt: sequences in the batch")
    ap.add_argument("--sp-split", default="block", choices=["block", "zigzag", "flat", "threshold"],
                    help="SP split rule of the destination layout (c4: DP4 x SP2)")
    ap.add_argument("--sp-min-len", type=int, default=8192, help="threshold split: shortest split sequence")
    ap.add_argument("--fields", default="scalar6-fp32+hidden2560")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-staged", action="store_true")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no clocks/e2e/cpu)")
    ap.add_argument("--exchange", choices=["p2p", "staged"], default="p2p",
                    help="N>1: fused P2P stores (default) or pack + grouped NCCL send/recv + unpack")
    ap.add_argument("--no-tune", action="store_true",
                    help="N>1: skip the pass that picks the NVLink store variant by measurement")
    return ap.parse_args()


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(desc):
    """DRAM bytes (read + write) of one copy_kernel launch from the committed ncu capture of the
    same workload (profiles/copy_kernel_traffic.json), else None."""
    p = os.path.join(ROOT, "profiles", "copy_kernel_traffic.json")
    try:
        d = json.load(open(p))
    except Exception:
        return None
    if d.get("workload") != desc:
        return None
    return int(d["dram_bytes_read"]) + int(d["dram_bytes_write"])


def workload(config, n_ranks, fields_name, n_seqs=512, sp_split="block", sp_min_len=0):
    from paper_2510_05943_b200 import workloads as W
    if config in ("c3", "c2-lpt"):
        lens = W.c2_lengths(0)
    elif config == "c0":  # fixed-overhead floor: the c3 layouts with every length 0
        lens = [0] * 512
    elif config == "c4":
        lens = W.c4_lengths(0)
    elif config == "c5":  # sweep series, uniform lengths, round-robin all-to-allv
        lens = [4096] * n_seqs
    else:  # c5-lt: sweep series with the C2 long-tail length distribution
        lens = W.lognormal_lengths(n_seqs, 2048, 0.75, 64, 8192, 0)
    import numpy as np
    lens = np.asarray(lens, dtype=np.int64)
    lay_cfg = {"c5-lt": "c5", "c0": "c3"}.get(config, config)
    src, dst = W.config_layouts(lay_cfg, n_ranks, len(lens))
    if sp_split != "block":
        dst = dict(dst, sp_split=sp_split, sp_min_len=sp_min_len if sp_split == "threshold" else 0)
    fields = W.field_set(fields_name)
    names = {
        "c3": "C2/C3 4B-class Tic-Tac-Toe batch: 512 episodes, lognormal(2048, 0.75) clip [64,8192]",
        "c0": "C0 fixed-overhead floor: 512 episodes of length 0",
        "c4": "C4 70B-class long context: 256 episodes, lognormal(8192, 0.6) clip [4096,32768]",
        "c2-lpt": "C2 batch, LPT rebalance",
        "c5": f"C5 uniform all-to-allv, {n_seqs} x L=4096",
        "c5-lt": f"C5 long-tail all-to-allv, {n_seqs} episodes lognormal(2048, 0.75) clip [64,8192]",
    }
    lay = lambda L: (f"DP{L['dp']}" + (f"xSP{L['sp']}" if L['sp'] > 1 else "")
                     + (f"({L['sp_split']})" if L.get("sp_split", "block") != "block" else "")
                     + (f"xTP{L['tp']}" if L['tp'] > 1 else "") + f"[{L['assign']}]")
    desc = f"{names[config]}; fields {fields_name}; {lay(src)} -> {lay(dst)}"
    return lens, src, dst, fields, desc


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 100 ms (B200_PROFILING.md clocks line)."""
    Q = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu=0):
        self.windows = []
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(gpu), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        time.sleep(0.6)

    def mark(self, t0, t1):
        self.windows.append((t0, t1))

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.25)
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        rows = []
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                ts = time.mktime(time.strptime(parts[0].split(".")[0], "%Y/%m/%d %H:%M:%S"))
                ts += float("0." + parts[0].split(".")[1]) if "." in parts[0] else 0.0
                rows.append((ts, float(parts[1]), float(parts[2]), parts[3:7]))
            except Exception:
                continue
        inwin = [r for r in rows if any(a - 0.15 <= r[0] <= b + 0.15 for a, b in self.windows)]
        use = inwin or rows
        if not use:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in use for k, v in enumerate(r[3]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[1] for r in use),
                "sm_max_mhz": max(r[2] for r in use), "reasons": reasons,
                "samples": len(use), "samples_in_timed_region": len(inwin)}


def nvlink_bytes(gpu):
    """Total NVLink data Tx and Rx bytes of one GPU from `nvidia-smi nvlink -gt d` (an independent
    cross-check of the plan's byte accounting); None when unavailable."""
    import re
    try:
        out = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", str(gpu)],
                             capture_output=True, text=True, timeout=20).stdout
    except Exception:
        return None
    tx = rx = 0
    seen = False
    for line in out.splitlines():
        m = re.search(r"(Tx|Rx)[^:]*:\s*([0-9]+)\s*(KiB|MiB|GiB|B)?", line)
        if not m:
            continue
        seen = True
        scale = {"KiB": 1024, "MiB": 1 << 20, "GiB": 1 << 30, "B": 1, None: 1024}[m.group(3)]
        if m.group(1) == "Tx":
            tx += int(m.group(2)) * scale
        else:
            rx += int(m.group(2)) * scale
    return (tx, rx) if seen else None


def emit(obj):
    print(json.dumps(obj), flush=True)


# ---------------------------------------------------------------------------------------
# CPU oracle (reference arm and cpu_baseline leg): the only places bench.py runs oracle/
# ---------------------------------------------------------------------------------------

def oracle_prepare(config, fields_name, n_seq_sample, seed=0):
    """Inputs for the oracle on the first n_seq_sample sequences of the workload, with the
    workload's layout shapes (8 ranks).  Payload bytes are random bits (the oracle moves
    opaque bytes; generating multi-GB float draws on the host would dominate the run)."""
    from oracle import earl_oracle as O
    from paper_2510_05943_b200 import workloads as W
    lens, _, _, fields, _ = workload(config, 8, fields_name)
    lens = [int(x) for x in lens[:n_seq_sample]]
    src, dst = W.config_layouts(config, 8, len(lens))
    glob = W.gen_global_fields(fields, sum(lens), seed_base=1000 + seed, random_bits=True)
    src_arrays = O.rank_arrays_from_global(src, lens, O.assign_groups(src, lens), glob, fields)
    del glob
    return (src, dst, lens, src_arrays, fields), sum(lens) * W.bytes_per_token(fields), sum(lens)


def oracle_core():
    """The core the oracle is pinned to (one core, reported): the first core of
    GPU 0's NUMA node when nvidia-smi reports its CPU affinity, else the first allowed core."""
    allowed = sorted(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else [0]
    try:
        out = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True,
                             timeout=20).stdout
        for line in out.splitlines():
            if line.startswith("GPU0"):
                for tok in line.split():
                    if "-" in tok and tok.replace("-", "").replace(",", "").isdigit():
                        first = int(tok.split(",")[0].split("-")[0])
                        if first in allowed:
                            return first
    except Exception:
        pass
    return allowed[0]


def oracle_run(prep):
    """Time the oracle's decentralized dispatch once, pinned to one
    core (the affinity is restored afterwards)."""
    from oracle import earl_oracle as O
    src, dst, lens, src_arrays, fields = prep
    old = os.sched_getaffinity(0) if hasattr(os, "sched_getaffinity") else None
    if old is not None:
        os.sched_setaffinity(0, {oracle_core()})
    try:
        t0 = time.perf_counter()
        O.dispatch(src, dst, lens, src_arrays, fields, 8)
        return time.perf_counter() - t0
    finally:
        if old is not None:
            os.sched_setaffinity(0, old)


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


REF_SEQS_PER_STEP = 32     # reference arm: bounded sample per step (~1 s of oracle work)
CPU_BASELINE_SEQS = 256    # cpu_baseline leg: ~10 s of oracle work


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    prep, nbytes, ntok = oracle_prepare(args.config, args.fields, REF_SEQS_PER_STEP)
    times = []
    for k in range(args.warmup + args.steps):
        dt = oracle_run(prep)
        if k >= args.warmup:
            times.append(dt)
    value = nbytes * len(times) / sum(times) / 1e9
    _, _, _, _, desc = workload(args.config, 8, args.fields)
    sample = (f"first {REF_SEQS_PER_STEP} sequences ({ntok} tokens, {nbytes} B) of the workload "
              f"per step, same layout shapes over 8 simulated ranks, single-threaded NumPy oracle")
    emit({"impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s",
          "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
          "ms_per_step": sum(times) / len(times) * 1e3, "higher_is_better": True,
          "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
          "config": {"workload": desc, "sample": sample},
          "cpu_baseline": {"value": value, "unit": "GB/s", "cores": 1, "kind": "oracle",
                           "pinned_core": oracle_core(),
                           "sample": sample},
          "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})


# ---------------------------------------------------------------------------------------
# N = 1: 8-rank emulation on one B200
# ---------------------------------------------------------------------------------------

def run_single(args):
    import numpy as np
    import torch

    from paper_2510_05943_b200 import earl
    from paper_2510_05943_b200 import workloads as W
    from paper_2510_05943_b200.dispatch import EmulatedDispatch

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    R = 8
    lens, src, dst, fields, desc = workload(args.config, R, args.fields, args.n_seqs, args.sp_split, args.sp_min_len)
    F = len(fields)
    Bf = [b * e for (_, b, e, _) in fields]
    ed = EmulatedDispatch(R)
    stream = torch.cuda.current_stream()
    lens_dev = torch.as_tensor(lens.astype(np.int32)).to(dev)

    # rollout-side holdings: each src rank's own tokens, drawn on the device
    counts = src["counts"]
    tok_r = W.rollout_token_counts(lens, counts)
    send = [W.gen_field_device(fields[f], tok_r[r], 1000 + 16 * r + f, dev)
            for r in range(R) for f in range(F)]
    plan = ed.plan(src, dst, lens_dev, fields)
    st = plan.stats()
    recv = ed.flat(ed.alloc_recv(plan, fields))
    stage = ed.alloc_stage(plan)
    plan.destroy()
    T, B = st["total_tokens"], st["bytes_per_token"]
    payload = T * B
    read_b = sum(st["read_bytes"])
    write_b = st["total"]
    alg_exec = read_b + write_b              # each source byte read once, written per replica
    alg_pack = 2 * read_b                    # read + write of every packed byte
    alg_unpack = read_b + write_b
    peak, peak_src = measured_peaks()

    # the plan object (device scratch) is made once; every step re-plans the batch on the
    # device (earl_plan_replan: header reset + planner) and dispatches it -- no allocation
    splan = ed.plan(src, dst, lens_dev, fields, stream)
    send_p, recv_p = earl.PtrArray(send), earl.PtrArray(recv)   # marshalled once (earl.PtrArray)

    def step(ev=None):
        if ev is not None:
            ev[0].record(stream)
        splan.replan(lens_dev, stream)
        if ev is not None:
            ev[1].record(stream)
        splan.exec(send_p, recv_p, stream)
        if ev is not None:
            ev[2].record(stream)

    clocks = None if args.profile else ClockSampler(0)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    launches0 = earl.kernel_launch_count()
    t0 = time.time()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    start.record(stream)
    for k in range(args.steps):
        step(evs[k])
    end.record(stream)
    torch.cuda.synchronize()
    t1 = time.time()
    launches = earl.kernel_launch_count() - launches0
    total_ms = start.elapsed_time(end)
    ms_step = total_ms / args.steps
    t_plan = statistics.median(e[0].elapsed_time(e[1]) for e in evs)
    t_exec = [e[1].elapsed_time(e[2]) for e in evs]
    t_exec_avg = sum(t_exec) / len(t_exec)
    if clocks:
        clocks.mark(t0, t1)

    out = {"metric": METRIC, "value": payload / (ms_step * 1e-3) / 1e9, "unit": "GB/s",
           "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
           "data": "synthetic (seeded device draws: ids uniform, logprobs -Exp(1), values/adv N(0,1),"
                   " mask Bernoulli(0.8), hidden N(0,1) bf16)",
           "config": {"workload": desc, "emulated_ranks": R, "global_batch": int(len(lens)),
                      "tokens": int(T), "bytes_per_token": int(B), "payload_bytes": int(payload),
                      "l2": "inputs larger than L2 (no flush needed)" if payload > 4 * 126e6
                      else "WARNING: payload fits in L2",
                      "parallelism": "8-rank emulation on 1 GPU"},
           "per_gpu_GBps": payload / (ms_step * 1e-3) / 1e9,
           "t_plan_ms": t_plan, "t_exec_ms": t_exec_avg,
           "roofline": {"bound": "hbm", "kernel": "copy_kernel (fused direct, all 8 ranks)",
                        "achieved": alg_exec / (t_exec_avg * 1e-3) / 1e9, "peak": peak,
                        "unit": "GB/s", "frac": alg_exec / (t_exec_avg * 1e-3) / 1e9 / peak,
                        "traffic": ncu_traffic(desc), "algorithmic_bytes": int(alg_exec),
                        "peak_source": peak_src},
           "gpu_launches": int(launches),
           "plan_stats": {"records": st["records"], "segments": st["segments"],
                          "read_bytes": int(read_b), "write_bytes": int(write_b)}}

    # the same step captured once as a CUDA graph (replan + exec) and replayed: the device-side
    # cost without host launch overhead (matters for the latency-bound small batches)
    if not args.profile:
        gs = torch.cuda.Stream()
        gs.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=gs):
            splan.replan(lens_dev, gs)
            splan.exec(send, recv, gs)
        for _ in range(args.warmup):
            graph.replay()
        torch.cuda.synchronize()
        ga, gb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ga.record(stream)
        for _ in range(args.steps):
            graph.replay()
        gb.record(stream)
        torch.cuda.synchronize()
        gms = ga.elapsed_time(gb) / args.steps
        out["graph"] = {"ms_per_step": gms, "value": payload / (gms * 1e-3) / 1e9,
                        "note": "replan + exec captured once as a CUDA graph, replayed per step"}
        del graph

    # staged path: plan + pack + unpack
    if not args.no_staged:
        ev2 = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
        for k in range(args.warmup + args.steps):
            e = ev2[k - args.warmup] if k >= args.warmup else None
            if e: e[0].record(stream)
            splan.replan(lens_dev, stream)
            if e: e[1].record(stream)
            splan.pack(send, stage, stream)
            if e: e[2].record(stream)
            splan.unpack(stage, recv, stream)
            if e: e[3].record(stream)
        ta = time.time()
        torch.cuda.synchronize()
        if clocks:
            clocks.mark(ta - 1e-3 * sum(x[0].elapsed_time(x[3]) for x in ev2), ta)
        tp = sum(x[1].elapsed_time(x[2]) for x in ev2) / args.steps
        tu = sum(x[2].elapsed_time(x[3]) for x in ev2) / args.steps
        tt = sum(x[0].elapsed_time(x[3]) for x in ev2) / args.steps
        out["staged"] = {
            "ms_per_step": tt, "value": payload / (tt * 1e-3) / 1e9,
            "pack": {"ms": tp, "achieved": alg_pack / (tp * 1e-3) / 1e9,
                     "frac": alg_pack / (tp * 1e-3) / 1e9 / peak, "algorithmic_bytes": int(alg_pack)},
            "unpack": {"ms": tu, "achieved": alg_unpack / (tu * 1e-3) / 1e9,
                       "frac": alg_unpack / (tu * 1e-3) / 1e9 / peak,
                       "algorithmic_bytes": int(alg_unpack)}}

    # end to end through the public API with host buffers (pinned), every step:
    # H2D of every source rank's payload + lengths, plan + exec, D2H of the destination metadata
    if not (args.no_e2e or args.profile):
        host_send = [torch.empty(t.numel(), dtype=torch.uint8, pin_memory=True) for t in send]
        for h, d in zip(host_send, send):
            h.copy_(d)
        lens_host = torch.as_tensor(lens.astype(np.int32)).pin_memory()
        dst_ranks = [r for r in range(R) if st["n_local_seqs"][r] > 0 or st["n_local_tokens"][r] > 0]
        metas = {r: torch.empty(int(st["n_local_seqs"][r]) + 1, dtype=torch.int32, device=dev)
                 for r in dst_ranks}
        meta_host = {r: torch.empty(m.numel(), dtype=torch.int32, pin_memory=True)
                     for r, m in metas.items()}
        h2d = sum(h.numel() for h in host_send) + lens_host.numel() * 4
        d2h = sum(m.numel() * 4 for m in metas.values())

        # the host-to-device copies run on a copy stream, one source rank after another; each
        # source's dispatch (earl_dispatch_exec_src) starts as soon as its bytes are resident,
        # so the copy engines and the SMs overlap (the copies still all sit in the timed region)
        copy_stream = torch.cuda.Stream(device=dev)
        ready = [torch.cuda.Event() for _ in range(R)]

        def e2e_step():
            lens_dev.copy_(lens_host, non_blocking=True)
            splan.replan(lens_dev, stream)
            copy_stream.wait_stream(stream)  # the previous step's dispatch has read `send`
            with torch.cuda.stream(copy_stream):
                for r in range(R):
                    for f in range(F):
                        send[r * F + f].copy_(host_send[r * F + f], non_blocking=True)
                    ready[r].record(copy_stream)
            for r in range(R):
                stream.wait_event(ready[r])
                splan.exec_src(r, send_p, recv_p, stream)
            for r in dst_ranks:
                splan.local_meta(r, metas[r], None, None, stream)
                meta_host[r].copy_(metas[r], non_blocking=True)

        n_e2e = max(3, min(args.steps, 10))
        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ta = time.time()
        a.record(stream)
        for _ in range(n_e2e):
            e2e_step()
        b.record(stream)
        torch.cuda.synchronize()
        if clocks:
            clocks.mark(ta, time.time())
        ems = a.elapsed_time(b) / n_e2e
        out["e2e"] = {"value": payload / (ems * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": ems,
                      "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                      "steps": n_e2e,
                      "path": "pinned host -> HBM per source rank on a copy stream, overlapped "
                              "with earl_dispatch_exec_src of the sources already resident"}
        del host_send

    if clocks:
        out["clocks"] = clocks.stop()

    if not (args.no_cpu_baseline or args.profile):
        prep, nbytes, ntok = oracle_prepare(args.config, args.fields, CPU_BASELINE_SEQS)
        dt = oracle_run(prep)
        del prep
        out["cpu_baseline"] = {
            "value": nbytes / dt / 1e9, "unit": "GB/s", "cores": 1, "kind": "oracle",
            "pinned_core": oracle_core(),
            "host_cores": os.cpu_count(), "affinity_cores": cpu_threads(), "seconds": dt,
            "sample": f"first {CPU_BASELINE_SEQS} sequences ({ntok} tokens, {nbytes} B) of the "
                      f"workload, same layout shapes over 8 simulated ranks; single-threaded "
                      f"NumPy oracle, random-bit payload"}
    emit(out)


# ---------------------------------------------------------------------------------------
# N > 1: one process per GPU
# ---------------------------------------------------------------------------------------

def run_multi(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2510_05943_b200 import earl
    from paper_2510_05943_b200 import workloads as W
    from paper_2510_05943_b200.dispatch import Dispatcher

    local = int(os.environ.get("LOCAL_RANK", "0"))
    # EARL_SHARED_GPU=1: every rank on cuda:0 with gloo plumbing -- validates the N>1 code path
    # on a one-GPU box (ranks time-slice the GPU, so its numbers are not performance numbers)
    shared = os.environ.get("EARL_SHARED_GPU") == "1"
    if shared:
        local = 0
    elif torch.cuda.device_count() <= local:
        raise SystemExit(f"bench.py --gpus {os.environ.get('WORLD_SIZE')}: rank {local} has no GPU "
                         f"({torch.cuda.device_count()} visible); EARL_SHARED_GPU=1 puts every "
                         "rank on cuda:0 (code-path check only)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if shared:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    rank, world = dist.get_rank(), dist.get_world_size()
    lens, src, dst, fields, desc = workload(args.config, world, args.fields, args.n_seqs, args.sp_split, args.sp_min_len)
    F = len(fields)
    B = W.bytes_per_token(fields)
    T = int(lens.sum())
    counts = src["counts"]
    tok_r = W.rollout_token_counts(lens, counts)
    edges = np.concatenate([[0], np.cumsum(counts)])
    my_lens = torch.as_tensor(lens[edges[rank]:edges[rank + 1]].astype(np.int32)).to(dev)
    send = [W.gen_field_device(fields[f], tok_r[rank], 1000 + 16 * rank + f, dev) for f in range(F)]
    D = Dispatcher(window_bytes=T * B + (1 << 20), device=local)
    stream = torch.cuda.current_stream()
    # step a1 on the device: the rollout's per-rank counts are fixed by the source layout, so the
    # length gather is one kernel over the peer windows (earl_allgather_lengths), no host sync
    from paper_2510_05943_b200.dispatch import rank_counts
    cnts = rank_counts(src, world)
    glens_buf = torch.empty(max(1, len(lens)), dtype=torch.int32, device=dev)
    glens, _ = D.allgather_lens(my_lens, counts=cnts, out=glens_buf)
    D.comm.check()
    assert glens.cpu().tolist() == [int(x) for x in lens], "a1: gathered lengths differ"
    plan = D.plan(src, dst, glens, fields)
    st = plan.stats()
    recv_ptrs, _views = D.alloc_recv(plan, fields)
    staged = args.exchange == "staged"
    plan.destroy()

    if staged and not shared:
        D.init_nccl()   # K8: the library's grouped ncclSend / ncclRecv (one GPU per rank)
    mplan = D.plan(src, dst, glens, fields, stream)
    send_p, recv_p = earl.PtrArray(send), earl.PtrArray(recv_ptrs)

    def step(ev=None):
        if ev is not None:
            ev[3].record(stream)
        gl, _ = D.allgather_lens(my_lens, counts=cnts, out=glens_buf, stream=stream)
        if ev is not None:
            ev[0].record(stream)
        p = mplan
        p.replan(gl, stream)
        if ev is not None:
            ev[1].record(stream)
        if staged:  # pack -> grouped NCCL send/recv -> unpack (the exchange comparator); the
            # per-peer byte table is read from the plan every step (a host sync NCCL needs)
            D.exec_staged(p, send, recv_ptrs, stream=stream)
        else:       # fused P2P: one pass, stores straight into the peers' windows
            p.exec(send_p, recv_p, stream)
        if ev is not None:
            ev[2].record(stream)

    # every rank samples its own GPU's clocks (shared-GPU mode: rank 0 only)
    clocks = ClockSampler(local) if (rank == 0 or not shared) and not args.profile else None
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    # choose the NVLink options by measurement (north_star: "whichever ... is faster"): peer
    # replicas by warp stores or TMA bulk stores, the default copy-engine shape or 8 warps;
    # every variant moves the same bytes, the fastest (max over ranks) is used for the timed loop
    tuning = None
    if not (staged or args.profile or args.no_tune):
        from paper_2510_05943_b200.dispatch import max_over_ranks as _mor
        variants = [(-1, -1), (1, -1), (0, 3), (1, 3)]
        times = []
        for rs, shape in variants:
            D.comm.set_exec_options(rs, shape)
            for _ in range(2):
                step()
            torch.cuda.synchronize()
            dist.barrier()
            ta_, tb_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ta_.record(stream)
            for _ in range(3):
                step()
            tb_.record(stream)
            torch.cuda.synchronize()
            times.append(_mor([ta_.elapsed_time(tb_) / 3])[0])
        best = min(range(len(variants)), key=lambda k: times[k])
        D.comm.set_exec_options(*variants[best])
        names = ["warp stores, default shape", "TMA stores, default shape",
                 "warp stores, 8 warps x 3 x 8 KB", "TMA stores, 8 warps x 3 x 8 KB"]
        tuning = {"ms_per_step": {names[k]: times[k] for k in range(len(variants))},
                  "chosen": names[best]}
        for _ in range(2):
            step()
        torch.cuda.synchronize()
        dist.barrier()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    nvl0 = nvlink_bytes(local) if not (shared or args.profile) else None
    l0 = earl.kernel_launch_count()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    a.record(stream)
    for k in range(args.steps):
        step(evs[k])
    b.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    t1 = time.time()
    launches = earl.kernel_launch_count() - l0
    from paper_2510_05943_b200.dispatch import max_over_ranks
    nvl1 = nvlink_bytes(local) if nvl0 is not None else None
    nvl_counted = None if (nvl0 is None or nvl1 is None) else \
        {"tx_bytes": nvl1[0] - nvl0[0], "rx_bytes": nvl1[1] - nvl0[1]}
    all_nvl = [None] * world
    dist.all_gather_object(all_nvl, nvl_counted)
    my_exec = sum(e[1].elapsed_time(e[2]) for e in evs) / args.steps
    ms_step, t_exec, t_plan, t_a1, neg_exec_min = max_over_ranks(
        [a.elapsed_time(b) / args.steps, my_exec,
         statistics.median(e[0].elapsed_time(e[1]) for e in evs),
         statistics.median(e[3].elapsed_time(e[0]) for e in evs), -my_exec])
    t_exec_min = -neg_exec_min
    clocks_r = None
    plan = D.plan(src, dst, glens, fields)
    plan.sync()
    plan.destroy()

    # end to end through the public API with host buffers: H2D of this rank's payload (pinned),
    # length all-gather, plan, exchange, D2H of this rank's cu_seqlens -- every step
    # the whole step (a1 gather + replan + exec) captured once as a CUDA graph and replayed
    graph_ms = None
    if not (args.profile or staged):
        gs = torch.cuda.Stream(device=dev)
        gs.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=gs):
            gl, _ = D.allgather_lens(my_lens, counts=cnts, out=glens_buf, stream=gs)
            mplan.replan(gl, gs)
            mplan.exec(send, recv_ptrs, gs)
        for _ in range(args.warmup):
            graph.replay()
        torch.cuda.synchronize()
        dist.barrier()
        ga, gb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ga.record(stream)
        for _ in range(args.steps):
            graph.replay()
        gb.record(stream)
        torch.cuda.synchronize()
        graph_ms = max_over_ranks([ga.elapsed_time(gb) / args.steps])[0]
        mplan.sync()
        del graph
    e2e = None
    if not (args.no_e2e or args.profile):
        host_send = [torch.empty(t.numel(), dtype=torch.uint8, pin_memory=True) for t in send]
        for hs, d in zip(host_send, send):
            hs.copy_(d)
        ns_mine = int(st["n_local_seqs"][rank])
        cu_dev = torch.empty(ns_mine + 1, dtype=torch.int32, device=dev)
        cu_host = torch.empty(ns_mine + 1, dtype=torch.int32, pin_memory=True)
        h2d = sum(hs.numel() for hs in host_send)

        my_lens_host = my_lens.cpu().pin_memory()
        h2d += my_lens_host.numel() * 4

        def e2e_step():
            for hs, d in zip(host_send, send):
                d.copy_(hs, non_blocking=True)
            my_lens.copy_(my_lens_host, non_blocking=True)
            gl, _ = D.allgather_lens(my_lens, counts=cnts, out=glens_buf, stream=stream)
            mplan.replan(gl, stream)
            if staged:
                D.exec_staged(mplan, send, recv_ptrs, stream=stream)
            else:
                mplan.exec(send_p, recv_p, stream)
            mplan.local_meta(rank, cu_dev, None, None, stream)
            cu_host.copy_(cu_dev, non_blocking=True)

        n_e2e = max(3, min(args.steps, 10))
        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        dist.barrier()
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record(stream)
        for _ in range(n_e2e):
            e2e_step()
        eb.record(stream)
        torch.cuda.synchronize()
        ems = max_over_ranks([ea.elapsed_time(eb) / n_e2e])[0]
        e2e = {"value": T * B / (ems * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": ems,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int((ns_mine + 1) * 4),
               "steps": n_e2e, "per_rank": True}
    if clocks:
        clocks.mark(t0, t1)
        clocks_r = clocks.stop()
    all_clocks = [None] * world
    dist.all_gather_object(all_clocks, clocks_r)
    mapped = sum(1 for p in range(world) if p != rank and D.comm.peer_mapped(p))
    all_mapped = [None] * world
    dist.all_gather_object(all_mapped, mapped)
    if rank == 0:
        payload = T * B
        nvl = max(max(st["egress"]), max(st["ingress"]))
        nvl_gbps = nvl / (t_exec * 1e-3) / 1e9
        out = {"metric": METRIC, "value": payload / (ms_step * 1e-3) / 1e9, "unit": "GB/s",
               "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
               "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
               "data": "synthetic (seeded device draws)",
               "config": {"workload": desc, "global_batch": int(len(lens)), "tokens": T,
                          "bytes_per_token": B, "payload_bytes": payload,
                          "l2": "inputs larger than L2", "parallelism": f"{world} ranks, P2P",
                          "shared_gpu": shared},
               "per_gpu_GBps": payload / (ms_step * 1e-3) / 1e9 / world,
               "t_a1_ms": t_a1, "t_plan_ms": t_plan, "t_exec_ms": t_exec,
               "t_exec_min_ms": t_exec_min,
               "exchange": args.exchange,
               "nvlink": {"bottleneck_bytes": int(nvl), "GBps": nvl_gbps,
                          "frac_measured_770": nvl_gbps / NVLINK_PEER_GBPS,
                          "frac_nominal_900": nvl_gbps / NVLINK_NOMINAL_GBPS,
                          "egress_per_rank": [int(x) for x in st["egress"]],
                          "ingress_per_rank": [int(x) for x in st["ingress"]],
                          "self_per_rank": [int(x) for x in st["self"]],
                          "note": "t_exec includes the entry barrier (rank skew): "
                                  "t_exec_ms is the max, t_exec_min_ms the min over ranks",
                          "nvidia_smi_counters_timed_region": all_nvl,
                          "plan_bytes_timed_region": {"egress_per_rank": [int(x) * args.steps for x in st["egress"]],
                                                      "ingress_per_rank": [int(x) * args.steps for x in st["ingress"]]}},
               "data_plane": {"kind": "CUDA IPC windows, fused P2P stores" if not staged
                              else ("pack + library NCCL grouped send/recv + unpack" if not shared
                                    else "pack + exchange over the gloo group + unpack"),
                              "mapped_peers_per_rank": all_mapped},
               "roofline": {"bound": "nvlink", "kernel": ("pack + NCCL send/recv + unpack" if staged
                                                          else "entry barrier + copy_kernel (P2P)"),
                            "achieved": nvl / (t_exec * 1e-3) / 1e9, "peak": NVLINK_PEER_GBPS,
                            "unit": "GB/s", "frac": nvl / (t_exec * 1e-3) / 1e9 / NVLINK_PEER_GBPS,
                            "traffic": None, "algorithmic_bytes": int(nvl),
                            "peak_source": "B200_PROFILING.md measured peer copy per direction"},
               "gpu_launches": int(launches) * world,
               "plan_stats": {"max_egress": st["max_egress"], "max_ingress": st["max_ingress"],
                              "moved": st["moved"], "records": st["records"]}}
        if e2e:
            out["e2e"] = e2e
        try:
            nccl_ver = ".".join(str(x) for x in torch.cuda.nccl.version())
        except Exception:
            nccl_ver = None
        out["comm"] = {"backend": dist.get_backend(), "nccl": nccl_ver,
                       "env": {k: v for k, v in sorted(os.environ.items()) if k.startswith("NCCL_")}}
        if graph_ms is not None:
            out["graph"] = {"ms_per_step": graph_ms, "value": payload / (graph_ms * 1e-3) / 1e9,
                            "note": "a1 gather + replan + exec captured once as a CUDA graph"}
        if tuning is not None:
            out["nvlink_options"] = tuning
        if all_clocks[0] is not None:
            c0 = dict(all_clocks[0])
            c0["per_rank"] = all_clocks
            out["clocks"] = c0
        emit(out)
    dist.barrier()
    dist.destroy_process_group()


def relaunch_under_torchrun(args):
    """`bench.py --gpus N` (N > 1) started without torchrun: re-execute this script under
    torch.distributed.run with one process per GPU (rank 0 prints the JSON line)."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    if world > 1:
        run_multi(args)
    else:
        run_single(args)


if __name__ == "__main__":
    main()
