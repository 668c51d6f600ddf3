export PYTHONUNBUFFERED=1
for i in 1 2 3 4 5 6; do timeout 300 python -m pytest tests/test_runtime_gpu.py::test_single_instance_prefetch_and_reuse -m gpu -q -x -p no:cacheprovider --tb=long > gpurun_out/flaky_$i.txt 2>&1; echo "try $i rc=$?"; done
timeout 300 python -m pytest tests/test_runtime_gpu.py -k cost_aware -m gpu -q -p no:cacheprovider --tb=short 2>&1 | tail -5
