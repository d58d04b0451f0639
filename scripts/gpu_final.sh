#!/bin/bash
# tests + tuning matrix (auto shape) + round artifacts
TAG=${TAG:-r01c}
bash scripts/gpu_round.sh
python scripts/tune.py "-1" "c3|c2-lpt|c4|c5-lt:131072:scalar6-fp32|c5:32768:scalar6-fp32|c3::scalar6-fp32" 2>&1 | tee gpurun_out/$TAG/matrix.txt
