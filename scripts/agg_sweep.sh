# returns_kernel compile-time knob sweep (C5-lt and C2 batches)
for cfg in "" "EARL_AGG_RING=3 EARL_AGG_CTAS_PER_SM=2" "EARL_AGG_RING=1" "EARL_AGG_RING=2 EARL_AGG_MAX_NB=16"; do
  EARL_NVCC_DEFINES="$cfg" python -m paper_2510_05943_b200.build > /dev/null 2>&1 || { echo "build failed: $cfg"; continue; }
  echo "== [$cfg]"
  python scripts/aggregate_bench.py 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    print('  %-26s returns %.3f ms (%.2f)  adv %.3f ms (%.2f)' % (d['workload'][:26], d['returns_ms'], d['returns_hbm_frac'], d['advantages_ms'], d['advantages_hbm_frac']))"
done
