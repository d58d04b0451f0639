#!/bin/bash
mkdir -p gpurun_out/r01
python -c "import __graft_entry__ as g; g.build()" || exit 1
for n in 2 4; do
  EARL_SHARED_GPU=1 timeout 600 torchrun --nnodes 1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2951$n \
     bench.py --gpus $n --steps 5 --warmup 2 --fields scalar6-fp32+hidden256 > gpurun_out/r01/shared_n$n.json 2> gpurun_out/r01/shared_n$n.err
  echo "shared n=$n rc=$?"; cat gpurun_out/r01/shared_n$n.json; tail -3 gpurun_out/r01/shared_n$n.err
done
for cfg in c5 c5-lt; do for n in 512 4096 32768 131072 400000; do
  timeout 300 python bench.py --config $cfg --n-seqs $n --fields scalar6-fp32 --steps 10 --warmup 3 --no-staged --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$cfg N=$n payload %.1f MB plan %.3f ms exec %.3f ms frac %.3f value %.0f GB/s' % (d['config']['payload_bytes']/1e6, d['t_plan_ms'], d['t_exec_ms'], d['roofline']['frac'], d['value']))"
done; done
