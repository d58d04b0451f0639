# returns_kernel: batches by TMA bulk copies into a per-warp 2-slot ring vs register loads
for cfg in "EARL_AGG_TMA=1" "EARL_AGG_TMA=1 EARL_AGG_CTAS_PER_SM=2" ""; do
  EARL_NVCC_DEFINES="$cfg" python -m paper_2510_05943_b200.build > /dev/null 2>&1 || { echo "build failed: $cfg"; continue; }
  echo "== [$cfg]"
  timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_multiprocess.py -m gpu -q -x -k "advantages or returns" 2>&1 | tail -1
  timeout 300 python scripts/aggregate_bench.py 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.rstrip()); continue
    print('  %-26s returns %.3f ms (%.3f)  adv %.3f ms (%.3f)' % (d['workload'][:26], d['returns_ms'], d['returns_hbm_frac'], d['advantages_ms'], d['advantages_hbm_frac']))"
done
python -m paper_2510_05943_b200.build > /dev/null 2>&1
