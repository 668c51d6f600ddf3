RDKV_LIB=paper_2504_11765_b200/_variants/librdkv_RDKV_ATTN_TRACE_1.so python scripts/micro/attn_tile_trace.py "$@" > /tmp/tr.txt 2>&1
sed -n '1,2p;8,14p;66,68p' /tmp/tr.txt; grep -A14 "^by-kind" /tmp/tr.txt
