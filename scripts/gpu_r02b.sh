OUT=gpurun_out/r02b; mkdir -p $OUT
free -g > $OUT/free.txt; nproc >> $OUT/free.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke.log
timeout 900 python -m pytest tests/test_gpu_a1_streams.py tests/test_multiprocess.py tests/test_bench_multi.py -q -x > $OUT/pytest_new.log 2>&1; echo "pytest new rc=$?"; tail -15 $OUT/pytest_new.log
timeout 900 python -m pytest tests/test_bench_parity.py -q -x > $OUT/pytest_parity.log 2>&1; echo "pytest parity rc=$?"; tail -15 $OUT/pytest_parity.log
