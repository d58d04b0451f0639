# ncu --set full (+ source) of returns_kernel on the C5-lt batch
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" >/dev/null
ncu --set full --clock-control none --import-source on -k regex:"returns_kernel" -s 3 -c 1 \
    -o gpurun_out/agg_ret_C5-lt -f python scripts/aggregate_bench.py --only C5-lt --iters 4 > gpurun_out/agg_ncu.log 2>&1
tail -2 gpurun_out/agg_ncu.log
