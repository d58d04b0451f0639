# TMA-ring returns_kernel: full GPU suite, sanitizers, aggregate numbers, SpeedOfLight
OUT=gpurun_out/r01h; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1200 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu.log
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_cases.py > $OUT/$tool.log 2>&1
  echo "== $tool"; grep -E "sanitize cases ok|ERROR SUMMARY|RACECHECK SUMMARY" $OUT/$tool.log | head -3
done
timeout 600 python scripts/aggregate_bench.py > $OUT/aggregate.jsonl 2>&1; cat $OUT/aggregate.jsonl
timeout 600 ncu --section SpeedOfLight --metrics l1tex__data_pipe_lsu_wavefronts.sum --clock-control none -k regex:"returns_kernel|advantage_kernel" -s 6 -c 2 python scripts/aggregate_bench.py --only C5-lt --iters 4 > $OUT/agg_sol.txt 2>&1
grep -E "returns_kernel|advantage_kernel|DRAM Throughput|L1/TEX Cache Throughput|Duration|wavefronts" $OUT/agg_sol.txt
