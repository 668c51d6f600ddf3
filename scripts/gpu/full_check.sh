# round-end rehearsal: smoke, the whole -m gpu suite, then the default bench (timed)
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
t0=$(date +%s); timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/fc_tests.log 2>&1; echo tests_rc=$? $(( $(date +%s)-t0 ))s
tail -3 gpurun_out/fc_tests.log
t0=$(date +%s); timeout 1500 python bench.py > gpurun_out/fc_bench.json 2> gpurun_out/fc_bench.err; echo bench_rc=$? $(( $(date +%s)-t0 ))s
tail -2 gpurun_out/fc_bench.err
