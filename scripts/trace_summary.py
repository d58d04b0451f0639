"""Summarise EARL_COPY_TRACE output: per launch, warp duration distribution and makespan."""
import statistics
import sys

launches, cur = [], None
for line in open(sys.argv[1]):
    if line.startswith("launch"):
        cur = []
        launches.append((line.strip(), cur))
    else:
        w, t0, t1, b, c = map(int, line.split())
        cur.append((w, t0, t1, b, c))
for name, rows in launches[-int(sys.argv[2]) if len(sys.argv) > 2 else 0:]:
    t0 = min(r[1] for r in rows)
    t1 = max(r[2] for r in rows)
    durs = sorted((r[2] - r[1]) / 1e3 for r in rows)
    starts = sorted((r[1] - t0) / 1e3 for r in rows)
    byt = sum(r[3] for r in rows)
    print(f"{name}: warps={len(rows)} makespan={(t1 - t0) / 1e3:.1f}us bytes={byt / 1e9:.3f}GB "
          f"dur p0={durs[0]:.1f} p10={durs[len(durs) // 10]:.1f} p50={statistics.median(durs):.1f} "
          f"p90={durs[9 * len(durs) // 10]:.1f} max={durs[-1]:.1f} | start max={starts[-1]:.1f}us "
          f"| chunks/warp p50={statistics.median(r[4] for r in rows)}")
