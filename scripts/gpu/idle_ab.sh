# A/B of the idle-warp skip in the attention softmax (decode: G valid rows of 128)
timeout 240 python -m pytest tests/test_decode_gpu.py -x -q 2>&1 | tail -1
timeout 300 python -m pytest tests/test_attention_gpu.py -x -q 2>&1 | tail -1
for r in 1 2; do
  echo "IDLE=1 $(timeout 200 python scripts/decode_ab.py 2>/dev/null | tail -1)"
  echo "IDLE=0 $(RDKV_LIB=paper_2504_11765_b200/_variants/librdkv_RDKV_ATTN_IDLE_0.so timeout 200 python scripts/decode_ab.py 2>/dev/null | tail -1)"
done
