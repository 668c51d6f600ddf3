set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s1_smoke.log 2>&1; echo smoke_rc=$?
t0=$(date +%s); timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s1_gputests.log 2>&1; echo gputests_rc=$? $(( $(date +%s)-t0 ))s
t0=$(date +%s); timeout 1200 python bench.py > gpurun_out/s1_bench.json 2> gpurun_out/s1_bench.err; echo bench_rc=$? $(( $(date +%s)-t0 ))s
tail -3 gpurun_out/s1_gputests.log
