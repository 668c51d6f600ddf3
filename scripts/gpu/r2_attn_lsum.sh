export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_attention_gpu.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
for rep in 1 2; do for v in 0 1; do echo -n "LSUM=$v C3: "; RDKV_LIB=paper_2504_11765_b200/_variants/librdkv_RDKV_ATTN_LSUM_$v.so python scripts/attn_perf.py --seqs 16 --new 64 --cached 5120 --dh 128 2>&1 | tail -1 | cut -c1-40; done; done
RDKV_LIB=paper_2504_11765_b200/_variants/librdkv_RDKV_ATTN_TRACE_1.so python scripts/micro/attn_tile_trace.py --seqs 16 --new 64 --cached 5120 --dh 128 2>&1 | grep -A3 "median per-tile"
