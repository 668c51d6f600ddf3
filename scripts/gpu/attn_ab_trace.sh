# attention A/B (scripts/gpu/attn_ab.sh) plus a per-tile trace of the default build's schedule at C3
bash scripts/gpu/attn_ab.sh "$@" 2>&1 | grep -v "^+"
RDKV_LIB=paper_2504_11765_b200/_variants/librdkv_RDKV_ATTN_TRACE_1.so python scripts/micro/attn_tile_trace.py --seqs 16 --new 64 --cached 5120 --dh 128 > /tmp/tr.txt 2>&1
sed -n '1,2p;8,14p;66,68p' /tmp/tr.txt
