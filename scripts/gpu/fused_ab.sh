timeout 900 python -m pytest tests/test_prefill_gpu.py tests/test_decode_gpu.py tests/test_gemm_gpu.py tests/test_parity_full_gpu.py tests/test_tp_gpu.py tests/test_runtime_gpu.py -x -q 2>&1 | tail -3
for v in 0 1; do
  echo "== RDKV_SMALLM_FUSED=$v"
  RDKV_SMALLM_FUSED=$v bash scripts/gpu/bench_quick.sh 2>&1 | grep -E "^decode|^ttft|^[0-9]" | cut -c1-330
done
