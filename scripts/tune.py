"""Copy-engine shape tuning: bench.py exec/pack/unpack fractions for EARL_COPY_CFG x workloads.
Usage: python scripts/tune.py "3 6 7" "c3|c5-lt:131072:scalar6-fp32|c5:32768:scalar6-fp32" """
import json
import os
import subprocess
import sys

cfgs = sys.argv[1].split()
works = sys.argv[2].split("|") if len(sys.argv) > 2 else ["c3", "c2-lpt", "c4", "c5-lt:131072:scalar6-fp32",
                                                           "c5:32768:scalar6-fp32", "c3::scalar6-fp32"]
for cfg in cfgs:
    for w in works:
        parts = w.split(":")
        args = ["--config", parts[0]]
        if len(parts) > 1 and parts[1]:
            args += ["--n-seqs", parts[1]]
        if len(parts) > 2 and parts[2]:
            args += ["--fields", parts[2]]
        if len(parts) > 3 and parts[3]:
            args += ["--sp-split", parts[3]]
        env = dict(os.environ, EARL_COPY_CFG=cfg)
        r = subprocess.run([sys.executable, "bench.py", "--steps", "10", "--warmup", "3", "--no-e2e",
                            "--no-cpu-baseline"] + args, capture_output=True, text=True, env=env)
        try:
            d = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception:
            print(f"cfg {cfg} {w}: FAILED {r.stderr[-500:]}")
            continue
        s = d.get("staged", {})
        print(f"cfg {cfg} {w:28s} | exec {d['t_exec_ms']:.3f} ms {d['roofline']['frac']:.3f} | "
              f"pack {s['pack']['ms']:.3f} {s['pack']['frac']:.3f} | unpack {s['unpack']['ms']:.3f} "
              f"{s['unpack']['frac']:.3f} | plan {d['t_plan_ms']:.3f} ms", flush=True)
