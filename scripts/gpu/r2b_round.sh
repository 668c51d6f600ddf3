export PYTHONUNBUFFERED=1
timeout 300 python tests/golden/make_gpu_blob.py 2>&1 | tail -2
timeout 300 python scripts/micro/nvls_probe.py > gpurun_out/nvls_probe.json 2>&1; tail -2 gpurun_out/nvls_probe.json
( time timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=900 --timeout-method=thread ) > gpurun_out/suite.txt 2>&1; echo "suite rc=$?"; tail -5 gpurun_out/suite.txt
( time timeout 1200 python bench.py ) > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_default.err
