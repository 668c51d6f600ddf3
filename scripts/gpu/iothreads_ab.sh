for r in 1 2; do
for t in 4 8 16 32; do
  echo "IO_THREADS=$t distinct $(RDKV_IO_THREADS=$t timeout 400 python scripts/micro/cold_path.py llama-3-8b 10 distinct 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k: round(v,1) for k,v in d["median"].items()})')"
done
done
