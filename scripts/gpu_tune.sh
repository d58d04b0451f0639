#!/bin/bash
# Parity tests, then the copy-engine shapes on the default workload and on a 1:1 workload.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for cfg in 0 1 2 3 4 5; do
  for extra in "--config c3" "--config c2-lpt" "--config c3 --fields scalar6-fp32"; do
    EARL_COPY_CFG=$cfg timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline $extra 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
s=d.get('staged',{})
print('cfg $cfg $extra', 'exec %.3f ms frac %.3f | pack %.3f ms %.3f | unpack %.3f ms %.3f | plan %.3f ms' % (d['t_exec_ms'], d['roofline']['frac'], s['pack']['ms'], s['pack']['frac'], s['unpack']['ms'], s['unpack']['frac'], d['t_plan_ms']))"
  done
done
