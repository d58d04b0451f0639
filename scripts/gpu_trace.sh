#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
for cfg in 0 5; do for c in c3 c2-lpt; do
  rm -f /tmp/tr.txt
  EARL_COPY_CFG=$cfg EARL_COPY_TRACE=/tmp/tr.txt timeout 300 python bench.py --steps 2 --warmup 1 --profile --no-staged --config $c > /dev/null 2>&1
  echo "cfg=$cfg config=$c"; python scripts/trace_summary.py /tmp/tr.txt 2
done; done
