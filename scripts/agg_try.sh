python -c "import __graft_entry__ as g; g.build()" >/dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_multiprocess.py -m gpu -q -x -k "advantages or returns" 2>&1 | tail -3
bash scripts/agg_sweep.sh 2>&1 | grep -E "==|C5-lt|C2|C4"
