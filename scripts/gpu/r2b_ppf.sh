export PYTHONUNBUFFERED=1
for v in 0 2 6 8; do echo "PPF=$v"; RDKV_LIB=paper_2504_11765_b200/_variants/librdkv_RDKV_ATTN_PPF_$v.so timeout 120 python scripts/attn_perf.py --seqs 16 --new 64 --cached 5120 --dh 128 2>&1 | tail -1; done
echo "PPF=4 (default)"; timeout 120 python scripts/attn_perf.py --seqs 16 --new 64 --cached 5120 --dh 128 2>&1 | tail -1
echo "non-PP"; RDKV_ATTN_PP=0 timeout 120 python scripts/attn_perf.py --seqs 16 --new 64 --cached 5120 --dh 128 2>&1 | tail -1
echo "PPF=4 cached 1024"; timeout 120 python scripts/attn_perf.py --seqs 16 --new 64 --cached 1024 --dh 128 2>&1 | tail -1
echo "non-PP cached 1024"; RDKV_ATTN_PP=0 timeout 120 python scripts/attn_perf.py --seqs 16 --new 64 --cached 1024 --dh 128 2>&1 | tail -1
