export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt
( time timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=900 --timeout-method=thread ) > gpurun_out/suite.txt 2>&1; echo "suite rc=$?"
tail -25 gpurun_out/suite.txt
( time timeout 1200 python bench.py ) > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_default.err
( time timeout 900 python bench.py --impl reference --steps 3 --warmup 3 ) > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 2 --warmup 1 --no-extras --no-serve > gpurun_out/ncu_bench.log 2>&1; echo "ncu rc=$?"
