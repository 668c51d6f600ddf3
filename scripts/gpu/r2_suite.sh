export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=600 --timeout-method=thread --deselect tests/test_parity_full_gpu.py > gpurun_out/suite.txt 2>&1; echo "suite rc=$?"
tail -15 gpurun_out/suite.txt
RDKV_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-extras --serve-queries 16 --serve-rates 12 > gpurun_out/r2_n2.json 2> gpurun_out/r2_n2.err; echo "n2 rc=$?"; tail -5 gpurun_out/r2_n2.err
