# NEXT-2 kernels: throughput + one ncu --set full capture each (C5-lt batch), into gpurun_out/r01g
OUT=gpurun_out/r01g; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python scripts/aggregate_bench.py > $OUT/aggregate.jsonl 2> $OUT/aggregate.err; cat $OUT/aggregate.jsonl
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"returns_kernel|advantage_kernel" -s 6 -c 2 \
   -o $OUT/aggregate_full -f python scripts/aggregate_bench.py --only C5-lt --iters 4 > $OUT/ncu_agg.log 2>&1; echo "ncu agg rc=$?"
python scripts/ncu_summary.py $OUT/aggregate_full.ncu-rep > $OUT/aggregate_ncu.txt 2>&1
timeout 600 ncu --section SpeedOfLight --clock-control none -k regex:"returns_kernel|advantage_kernel" -s 6 -c 2 python scripts/aggregate_bench.py --only C5-lt --iters 4 > $OUT/agg_sol.txt 2>&1
rm -f $OUT/aggregate_full.ncu-rep
