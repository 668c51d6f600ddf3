export PYTHONUNBUFFERED=1
RDKV_ATTN_PP=1 RDKV_ATTN_SPL=2 timeout 600 python -m pytest tests/test_attention_gpu.py -m gpu -q -x -p no:cacheprovider -k "not stream_k" 2>&1 | tail -4
for cfg in "RDKV_ATTN_PP=1 RDKV_ATTN_SPL=2" "RDKV_ATTN_PP=1" "RDKV_ATTN_PP=0"; do echo "$cfg"; env $cfg timeout 120 python scripts/attn_perf.py --seqs 16 --new 64 --cached 5120 --dh 128 2>&1 | tail -1; env $cfg timeout 120 python scripts/attn_perf.py --seqs 16 --new 64 --cached 5120 --dh 128 --same-block 2>&1 | tail -1; done
