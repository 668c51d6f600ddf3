export PYTHONUNBUFFERED=1
timeout 300 python tests/golden/make_gpu_blob.py gpurun_out/gpu_store 2>&1 | tail -2
timeout 600 python -m pytest tests/test_runtime_gpu.py -m gpu -q -x -p no:cacheprovider --timeout=500 --timeout-method=thread 2>&1 | tail -3
timeout 300 python scripts/micro/disk_read.py > gpurun_out/disk_read.json 2>&1; cat gpurun_out/disk_read.json
df -h /tmp . | tail -2
