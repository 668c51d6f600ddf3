export PYTHONUNBUFFERED=1
timeout 900 python bench.py --model llama-3.2-1b --k 5 --batch 32 --steps 10 --warmup 3 > gpurun_out/r2_bench_c2.json 2> gpurun_out/r2_bench_c2.err; echo "c2 rc=$?"; tail -2 gpurun_out/r2_bench_c2.err
RDKV_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-extras --serve-queries 16 --serve-rates 12 > gpurun_out/r2_bench_n2_shared.json 2> gpurun_out/r2_bench_n2_shared.err; echo "n2 rc=$?"; tail -3 gpurun_out/r2_bench_n2_shared.err
