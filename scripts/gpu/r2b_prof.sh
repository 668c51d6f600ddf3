export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_runtime_gpu.py -m gpu -q -p no:cacheprovider --timeout=500 --timeout-method=thread 2>&1 | tail -3
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_c3_step_launches.csv python scripts/prof_step.py --steps 2 > gpurun_out/prof_launch.log 2>&1; echo "launch rc=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -s 12 -c 8 -o gpurun_out/r2_c3_layer python scripts/prof_step.py --steps 1 --graph 0 > gpurun_out/prof_full.log 2>&1; echo "full rc=$?"
timeout 1200 python scripts/c5_full.py > gpurun_out/r2_c5_full_depth.json 2> gpurun_out/c5.err; echo "c5 rc=$?"; tail -3 gpurun_out/c5.err; head -c 600 gpurun_out/r2_c5_full_depth.json
