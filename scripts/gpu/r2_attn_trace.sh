RDKV_LIB=paper_2504_11765_b200/_variants/librdkv_RDKV_ATTN_TRACE_1.so python scripts/micro/attn_tile_trace.py --seqs 16 --new 64 --cached 5120 --dh 128 2>&1 | tail -70
