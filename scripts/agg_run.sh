set -e
python -c "import __graft_entry__ as g; g.build()" >/dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_multiprocess.py -m gpu -q -x -k "advantages or returns" 2>&1 | tail -3
python scripts/aggregate_bench.py 2>&1 | tail -3
if [ -n "$AGG_NCU" ]; then
  ncu --set full --clock-control none --import-source on -k regex:"returns_kernel" -s 3 -c 1 \
      -o gpurun_out/agg_ret_C5-lt -f python scripts/aggregate_bench.py --only C5-lt --iters 4 > gpurun_out/agg_ncu.log 2>&1
  tail -1 gpurun_out/agg_ncu.log
fi
