export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_attention_gpu.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
for lib in "" "RDKV_LIB=paper_2504_11765_b200/_variants/librdkv_RDKV_ATTN_SPLITKV_0.so"; do echo "lib=$lib";
env $lib timeout 120 python scripts/attn_perf.py --seqs 16 --new 64 --cached 5120 --dh 128 2>&1 | tail -1
env $lib timeout 120 python scripts/attn_perf.py --seqs 32 --new 64 --cached 2560 --dh 64 2>&1 | tail -1
env $lib timeout 120 python scripts/attn_perf.py --seqs 1 --new 5184 --cached 0 --dh 128 2>&1 | tail -1
done
