timeout 600 python -m pytest tests/test_store_gpu.py tests/test_store.py tests/test_prefill_gpu.py tests/test_runtime_gpu.py -x -q 2>&1 | tail -2
for r in 1 2; do
  for s in 1 0; do
    echo "STREAM=$s distinct $(RDKV_STREAM_READ=$s timeout 400 python scripts/micro/cold_path.py llama-3-8b 10 distinct 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k: round(v,1) for k,v in d["median"].items()})')"
  done
done
