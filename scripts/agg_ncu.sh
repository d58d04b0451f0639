# ncu --set full of returns_kernel / advantage_kernel on the C2 batch and the C5-lt batch
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" >/dev/null
for w in C2 C5-lt; do
  ncu --set full --clock-control none --import-source on -k regex:"returns_kernel|advantage_kernel" -s 6 -c 2 \
      -o gpurun_out/agg_${w} -f python scripts/aggregate_bench.py --only "$w" --iters 4 > gpurun_out/agg_ncu_${w}.log 2>&1
  tail -3 gpurun_out/agg_ncu_${w}.log
done
