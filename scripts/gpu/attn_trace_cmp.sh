# per-tile trace summaries of the C3 attention shape vs an L2-resident KV set and a half grid
export RDKV_LIB=paper_2504_11765_b200/_variants/librdkv_RDKV_ATTN_TRACE_1.so
for args in "--seqs 16 --new 64 --cached 5120" "--seqs 16 --new 64 --cached 1024" "--seqs 8 --new 64 --cached 5120" "--seqs 16 --new 64 --cached 5120 --same-block"; do
  echo "=== $args"
  python scripts/micro/attn_tile_trace.py $args --dh 128 > /tmp/tr.txt 2>&1
  head -1 /tmp/tr.txt; grep -A0 "median" /tmp/tr.txt
  echo "producer rows 10-13:"; grep -A80 "^producer" /tmp/tr.txt | sed -n 12,15p
  echo "issuer rows 10-13:"; grep -A80 "^issuer 0" /tmp/tr.txt | sed -n 11,14p
done
