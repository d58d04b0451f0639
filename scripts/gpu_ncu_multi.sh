#!/bin/bash
# Several full ncu captures of copy_kernel: TAG:CFG:bench-args triples separated by ';'
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
IFS=';' read -ra RUNS <<< "$1"
for run in "${RUNS[@]}"; do
  TAG=$(echo $run | cut -d: -f1); CFG=$(echo $run | cut -d: -f2); ARGS=$(echo $run | cut -d: -f3)
  EARL_COPY_CFG=$CFG timeout 900 ncu --set full --clock-control none --import-source on -k regex:copy_kernel -s 1 -c 1 \
    -o gpurun_out/prof_$TAG -f python bench.py --steps 2 --warmup 1 --profile --no-staged $ARGS > gpurun_out/ncu_$TAG.log 2>&1
  echo "$TAG rc=$?"
done
