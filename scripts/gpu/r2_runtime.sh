set -x
timeout 900 python -m pytest tests/test_runtime_gpu.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -30
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --deselect tests/test_parity_full_gpu.py 2>&1 | tail -15
