export PYTHONUNBUFFERED=1
df -h /tmp /dev/shm | tee gpurun_out/df.txt
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_c3_c.json 2> gpurun_out/r2_c3_c.err; echo "bench rc=$?"; tail -3 gpurun_out/r2_c3_c.err
timeout 600 python -m pytest tests/test_runtime_gpu.py -m gpu -x -q -p no:cacheprovider --timeout=300 --timeout-method=thread 2>&1 | tail -5
