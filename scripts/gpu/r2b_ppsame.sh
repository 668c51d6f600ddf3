export PYTHONUNBUFFERED=1
for pp in 1 0; do echo "PP=$pp same-block"; RDKV_LIB=paper_2504_11765_b200/_variants/librdkv_RDKV_ATTN_PPF_0.so RDKV_ATTN_PP=$pp timeout 120 python scripts/attn_perf.py --seqs 16 --new 64 --cached 5120 --dh 128 --same-block 2>&1 | tail -1; done
