# round-end rehearsal: smoke, the whole -m gpu suite, the default bench, the reference arm, ncu evidence
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
t0=$(date +%s); timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final_tests.log 2>&1; echo tests_rc=$? $(( $(date +%s)-t0 ))s
tail -2 gpurun_out/final_tests.log
t0=$(date +%s); timeout 1500 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo bench_rc=$? $(( $(date +%s)-t0 ))s
t0=$(date +%s); timeout 900 python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo ref_rc=$? $(( $(date +%s)-t0 ))s
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --profile-from-start off --csv --log-file gpurun_out/final_step_launches.csv python scripts/prof_step.py --steps 2 > /dev/null 2>&1; echo ncu_step=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --profile-from-start off --csv --log-file gpurun_out/final_decode_launches.csv python scripts/prof_decode.py 2 > /dev/null 2>&1; echo ncu_decode=$?
