#!/bin/bash
# Round artifacts on one B200: tests, smoke, bench (ours + reference), ncu launch list and one
# full ncu capture of the copy kernel.  Everything lands in gpurun_out/$TAG/.
TAG=${TAG:-r01}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke.log
timeout 1200 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; cat $OUT/bench.json
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?"; cat $OUT/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
   python bench.py --steps 5 --warmup 2 --profile > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:copy_kernel -s 1 -c 1 \
   -o $OUT/copy_full -f python bench.py --steps 2 --warmup 1 --profile --no-staged > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
# NEXT-2: distributed returns / advantages (C2, C4, C5-lt batches) and one full capture each
timeout 600 python scripts/aggregate_bench.py > $OUT/aggregate.jsonl 2> $OUT/aggregate.err; echo "aggregate rc=$?"; cat $OUT/aggregate.jsonl
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"returns_kernel|advantage_kernel" -s 6 -c 2 \
   -o $OUT/aggregate_full -f python scripts/aggregate_bench.py --only C5-lt --iters 4 > $OUT/ncu_agg.log 2>&1; echo "ncu agg rc=$?"
