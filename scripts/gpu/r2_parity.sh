set -x
python -m pytest tests/test_oracle_hf.py tests/test_parity_full_gpu.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -15
python -m pytest tests/test_prefill_gpu.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
python bench.py --steps 5 --warmup 3 > gpurun_out/r2_c3_b.json 2> gpurun_out/r2_c3_b.err; tail -3 gpurun_out/r2_c3_b.err
