export PYTHONUNBUFFERED=1
RDKV_LIB=paper_2504_11765_b200/_variants/librdkv_RDKV_ATTN_TRACE_1.so timeout 300 python scripts/micro/attn_tile_trace.py --seqs 16 --new 64 --cached 5120 --dh 128 > gpurun_out/attn_trace_pp.txt 2>&1; head -45 gpurun_out/attn_trace_pp.txt
