#!/bin/bash
# Round artifacts on one B200: smoke, pytest -m gpu, bench (ours + reference arm, N = 1), the
# N = 2 path on one GPU (EARL_SHARED_GPU=1, code path only), the ncu launch list and one full
# ncu capture of the copy kernel, the planner profile, the C5 sweep, the NEXT-2 aggregate bench
# and its capture.  Everything lands in gpurun_out/$TAG/.
TAG=${TAG:-r02}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; cat $OUT/bench.json
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?"; cat $OUT/bench_ref.json
EARL_SHARED_GPU=1 timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_n2_shared.json 2> $OUT/bench_n2.err; echo "n2 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
   python bench.py --steps 5 --warmup 2 --profile > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
python scripts/launch_summary.py $OUT/launches.csv > $OUT/launches_summary.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:copy_kernel -s 1 -c 1 \
   -o $OUT/copy_full -f python bench.py --steps 2 --warmup 1 --profile --no-staged > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
python scripts/ncu_summary.py $OUT/copy_full.ncu-rep > $OUT/copy_ncu.txt 2>&1
REPS=20 timeout 300 python scripts/plan_profile.py > $OUT/plan_profile.jsonl 2>&1
timeout 1200 python scripts/sweep.py $TAG > $OUT/sweep.jsonl 2>&1; echo "sweep rc=$?"; cp gpurun_out/${TAG}_sweep.* $OUT/ 2>/dev/null
timeout 600 python scripts/aggregate_bench.py > $OUT/aggregate.jsonl 2> $OUT/aggregate.err; echo "aggregate rc=$?"; cat $OUT/aggregate.jsonl
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"returns_units_kernel|advantage_kernel" -s 4 -c 2 \
   -o $OUT/aggregate_full -f python scripts/aggregate_bench.py --only C5-lt --iters 4 > $OUT/ncu_agg.log 2>&1; echo "ncu agg rc=$?"
python scripts/ncu_summary.py $OUT/aggregate_full.ncu-rep > $OUT/aggregate_ncu.txt 2>&1
rm -f $OUT/*.ncu-rep.tmp
ls $OUT
