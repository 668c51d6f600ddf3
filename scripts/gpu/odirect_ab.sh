# cold-disk read: buffered parallel pread vs O_DIRECT (RDKV_ODIRECT=1), C3 640-MiB composites
for r in 1 2; do
  for d in 0 1; do
    echo "ODIRECT=$d distinct $(RDKV_ODIRECT=$d timeout 400 python scripts/micro/cold_path.py llama-3-8b 10 distinct 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["median"])')"
  done
done
for d in 0 1; do
  echo "ODIRECT=$d reread $(RDKV_ODIRECT=$d timeout 400 python scripts/micro/cold_path.py llama-3-8b 10 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["median"])')"
done
RDKV_ODIRECT=1 timeout 300 python -m pytest tests/test_store.py tests/test_prefill_gpu.py -q -x -k "not aligned" 2>&1 | tail -1
