#!/bin/bash
# Parity, then exec/pack/unpack fractions over workloads for the copy-engine shapes in $CFGS.
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for cfg in ${CFGS:-0 1 3}; do
  for extra in ${EXTRAS:-"--config c3" "--config c2-lpt" "--config c4" "--config c5-lt --n-seqs 131072 --fields scalar6-fp32" "--config c5 --n-seqs 32768 --fields scalar6-fp32" "--config c3 --fields scalar6-fp32"}; do
    EARL_COPY_CFG=$cfg timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $extra 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
s=d.get('staged',{})
print('cfg $cfg $extra', '| exec %.3f ms %.3f | pack %.3f ms %.3f | unpack %.3f ms %.3f | plan %.3f ms' % (d['t_exec_ms'], d['roofline']['frac'], s['pack']['ms'], s['pack']['frac'], s['unpack']['ms'], s['unpack']['frac'], d['t_plan_ms']))"
  done
done
