# correctness of the default build on the GEMM / decode tests, then bench_quick per lib
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_decode_gpu.py tests/test_prefill_gpu.py -x -q 2>&1 | tail -1
for lib in "$@"; do
  echo "== $lib"
  RDKV_LIB=$lib bash scripts/gpu/bench_quick.sh 2>&1 | grep -E "^decode|^ttft|^[0-9]" | cut -c1-230
done
