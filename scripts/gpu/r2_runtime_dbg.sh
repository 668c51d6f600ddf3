export PYTHONUNBUFFERED=1 RDKV_RT_DEBUG=1
timeout 250 python -m pytest tests/test_runtime_gpu.py -m gpu -x -q -s -p no:cacheprovider --timeout=100 --timeout-method=thread -k single > gpurun_out/rt_dbg1.txt 2>&1
timeout 250 python -m pytest tests/test_runtime_gpu.py -m gpu -x -q -s -p no:cacheprovider --timeout=200 --timeout-method=thread -k two > gpurun_out/rt_dbg2.txt 2>&1
