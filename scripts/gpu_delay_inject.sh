# Delay injection (EARL_DELAY_INJECT=1: pseudo-random spins at the entry barrier, the copy
# kernel's start and completion protocol, the returns look-back publication and the planner's
# grid barriers): the timing-sensitive GPU tests must stay bit-exact / within bound.
OUT=gpurun_out/delay; mkdir -p $OUT
EARL_NVCC_DEFINES="EARL_DELAY_INJECT=1" python -m paper_2510_05943_b200.build > $OUT/build.log 2>&1 || { echo "build failed"; exit 1; }
timeout 2400 python -m pytest tests/test_multiprocess.py tests/test_gpu_parity.py tests/test_gpu_a1_streams.py -m gpu -q \
  -k "processes or returns or advantages or large_n or random_layouts or cooperative or replan or graph or exec_src or null_recv or late_peer or variants or gather or streams or fast_planner" \
  > $OUT/pytest.log 2>&1; echo "delay-injected pytest rc=$?"; tail -1 $OUT/pytest.log
python -m paper_2510_05943_b200.build > /dev/null 2>&1
