for rep in 1 2; do
for v in 2 3 4; do echo -n "ST128=$v C3: "; RDKV_LIB=paper_2504_11765_b200/_variants/librdkv_RDKV_ATTN_ST128_$v.so python scripts/attn_perf.py --seqs 16 --new 64 --cached 5120 --dh 128 2>&1 | tail -1 | cut -c1-40; done
for v in 3 4 5; do echo -n "ST64=$v C2: "; RDKV_LIB=paper_2504_11765_b200/_variants/librdkv_RDKV_ATTN_ST64_$v.so python scripts/attn_perf.py --seqs 32 --new 64 --cached 2560 --dh 64 2>&1 | tail -1 | cut -c1-40; done
done
