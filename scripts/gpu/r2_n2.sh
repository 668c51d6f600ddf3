export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_sanitizer_gpu.py tests/test_serving_gpu.py -m gpu -q -p no:cacheprovider --timeout=500 --timeout-method=thread 2>&1 | tail -3
RDKV_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-extras --serve-queries 16 --serve-rates 12 > gpurun_out/r2_n2.json 2> gpurun_out/r2_n2.err; echo "n2 rc=$?"; grep -v Warning gpurun_out/r2_n2.err | tail -5
