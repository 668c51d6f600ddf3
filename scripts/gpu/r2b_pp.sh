export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_attention_gpu.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -15
for pp in 1 0; do RDKV_ATTN_PP=$pp timeout 120 python scripts/attn_perf.py --seqs 16 --new 64 --cached 5120 --dh 128 2>&1 | tail -1; done
for pp in 1 0; do RDKV_ATTN_PP=$pp timeout 120 python scripts/attn_perf.py --seqs 1 --new 64 --cached 5120 --dh 128 2>&1 | tail -1; done
for pp in 1 0; do RDKV_ATTN_PP=$pp timeout 120 python scripts/attn_perf.py --seqs 1 --new 5184 --cached 0 --dh 128 2>&1 | tail -1; done
