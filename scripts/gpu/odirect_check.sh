timeout 900 python -m pytest tests/test_store.py tests/test_runtime_gpu.py tests/test_serving_gpu.py tests/test_prefill_gpu.py tests/test_gpu_fixture.py tests/test_store_oplog.py -x -q 2>&1 | tail -2
bash scripts/gpu/bench_quick.sh
