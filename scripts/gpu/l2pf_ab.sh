timeout 600 python -m pytest tests/test_attention_gpu.py tests/test_gemm_gpu.py tests/test_prefill_gpu.py tests/test_decode_gpu.py -x -q 2>&1 | tail -1
for v in 0 1; do
  echo "== RDKV_SMALLM_L2PF=$v"
  RDKV_SMALLM_L2PF=$v bash scripts/gpu/bench_quick.sh 2>&1 | grep -E "^decode|^ttft|^[0-9]" | cut -c1-260
done
