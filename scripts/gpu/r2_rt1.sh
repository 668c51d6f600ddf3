export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_runtime_gpu.py -m gpu -x -q -p no:cacheprovider --timeout=200 --timeout-method=thread 2>&1 | grep -v "^  File\|^    " | tail -40 > gpurun_out/rt1.txt
