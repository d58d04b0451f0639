#!/bin/bash
# Iteration check: parity tests, trace of stragglers, and the copy-engine shapes.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for cfg in ${CFGS:-0 1 3 5}; do for c in c3 c2-lpt; do
  rm -f /tmp/tr.txt
  EARL_COPY_CFG=$cfg EARL_COPY_TRACE=/tmp/tr.txt timeout 300 python bench.py --steps 2 --warmup 1 --profile --no-staged --config $c > /dev/null 2>&1
  echo "cfg=$cfg config=$c"; python scripts/trace_summary.py /tmp/tr.txt 1
done; done
for cfg in ${CFGS:-0 1 3 5}; do
  for extra in "--config c3" "--config c2-lpt" "--config c4" "--config c3 --fields scalar6-fp32"; do
    EARL_COPY_CFG=$cfg timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline $extra 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
s=d.get('staged',{})
print('cfg $cfg $extra', 'exec %.3f ms frac %.3f | pack %.3f ms %.3f | unpack %.3f ms %.3f | plan %.3f ms' % (d['t_exec_ms'], d['roofline']['frac'], s['pack']['ms'], s['pack']['frac'], s['unpack']['ms'], s['unpack']['frac'], d['t_plan_ms']))"
  done
done
