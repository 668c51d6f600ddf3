export PYTHONUNBUFFERED=1
for c in 5120 1024; do
python scripts/attn_perf.py --seqs 16 --new 64 --cached $c --dh 128 2>&1 | tail -1
RDKV_LIB=paper_2504_11765_b200/_variants/librdkv_RDKV_ATTN_TRACE_1.so timeout 300 python scripts/micro/attn_tile_trace.py --seqs 16 --new 64 --cached $c --dh 128 > gpurun_out/attn_trace_c3_$c.txt 2>&1; grep -A3 "median per-tile" gpurun_out/attn_trace_c3_$c.txt
done
timeout 600 python scripts/gemm_c3.py > gpurun_out/r2_gemm_c3b.txt 2>&1; cat gpurun_out/r2_gemm_c3b.txt
for i in 1 2 3; do timeout 600 python -m pytest tests/test_runtime_gpu.py::test_single_instance_prefetch_and_reuse -m gpu -x -q -p no:cacheprovider --timeout=500 --timeout-method=thread > gpurun_out/rt_try$i.txt 2>&1; echo "rt$i rc=$?"; done
