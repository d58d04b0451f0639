#!/bin/bash
# Full ncu capture of the hot kernel (one launch), 1 GPU.  Usage: scripts/gpu_ncu_full.sh TAG [bench args]
TAG=$1; shift
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:copy_kernel -s 1 -c 1 \
  -o gpurun_out/prof_$TAG -f python bench.py --steps 2 --warmup 1 --profile --no-staged "$@" > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?"; tail -5 gpurun_out/ncu_$TAG.log
ls -la gpurun_out/
