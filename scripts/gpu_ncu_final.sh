OUT=gpurun_out/r01n; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
   python bench.py --steps 5 --warmup 2 --profile > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:copy_kernel -s 1 -c 1 \
   -o $OUT/copy_full -f python bench.py --steps 2 --warmup 1 --profile --no-staged > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
python scripts/launch_summary.py $OUT/launches.csv > $OUT/launches_summary.txt 2>&1
python scripts/ncu_summary.py $OUT/copy_full.ncu-rep > $OUT/copy_ncu.txt 2>&1
ncu -i $OUT/copy_full.ncu-rep --page raw --csv > $OUT/copy_raw.csv 2>/dev/null
rm -f $OUT/copy_full.ncu-rep
cat $OUT/launches_summary.txt; head -8 $OUT/copy_ncu.txt
