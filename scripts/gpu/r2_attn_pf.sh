export PYTHONUNBUFFERED=1
for rep in 1 2; do
for v in 0 2 4 6 8; do
  echo -n "PF=$v C3: "; RDKV_LIB=paper_2504_11765_b200/_variants/librdkv_RDKV_ATTN_PF_$v.so python scripts/attn_perf.py --seqs 16 --new 64 --cached 5120 --dh 128 2>&1 | tail -1 | cut -c1-60
  echo -n "PF=$v C2: "; RDKV_LIB=paper_2504_11765_b200/_variants/librdkv_RDKV_ATTN_PF_$v.so python scripts/attn_perf.py --seqs 32 --new 64 --cached 2560 --dh 64 2>&1 | tail -1 | cut -c1-60
done; done
