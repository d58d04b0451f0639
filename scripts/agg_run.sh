set -e
python -c "import __graft_entry__ as g; g.build()" >/dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_multiprocess.py -m gpu -q -x -k "advantages or returns" 2>&1 | tail -3
python scripts/aggregate_bench.py 2>&1 | tail -3
