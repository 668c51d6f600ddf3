export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout=600 --timeout-method=thread > gpurun_out/suite2.txt 2>&1; echo "suite rc=$?"; tail -12 gpurun_out/suite2.txt
timeout 900 python bench.py --steps 5 --warmup 3 --no-serve > gpurun_out/r2_c3_d.json 2> gpurun_out/r2_c3_d.err; echo "bench rc=$?"; tail -3 gpurun_out/r2_c3_d.err
