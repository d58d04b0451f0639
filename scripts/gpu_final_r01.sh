#!/bin/bash
# Round-1 refresh of every judged artifact on one B200, into gpurun_out/r01f/
TAG=r01f bash scripts/gpu_round.sh
python scripts/launch_summary.py gpurun_out/r01f/launches.csv > gpurun_out/r01f/launches_summary.txt 2>&1
python scripts/ncu_summary.py gpurun_out/r01f/copy_full.ncu-rep > gpurun_out/r01f/copy_ncu.txt 2>&1
python scripts/ncu_summary.py gpurun_out/r01f/aggregate_full.ncu-rep > gpurun_out/r01f/aggregate_ncu.txt 2>&1
ncu -i gpurun_out/r01f/copy_full.ncu-rep --page raw --csv > gpurun_out/r01f/copy_raw.csv 2>/dev/null
rm -f gpurun_out/r01f/*.ncu-rep.tmp
ls -la gpurun_out/r01f
