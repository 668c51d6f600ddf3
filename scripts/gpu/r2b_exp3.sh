export PYTHONUNBUFFERED=1
RDKV_LIB=paper_2504_11765_b200/_variants/librdkv_RDKV_ATTN_TRACE_1.so timeout 300 python scripts/micro/attn_tile_trace.py --seqs 16 --new 64 --cached 5120 --dh 128 > gpurun_out/attn_trace_c3_iss.txt 2>&1; grep -A70 "issuer 0 per tile" gpurun_out/attn_trace_c3_iss.txt | head -70
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_prefill_gpu.py tests/test_parity_full_gpu.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
