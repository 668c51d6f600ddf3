for s in 1 0 1 0; do
  RDKV_STREAM_READ=$s RDKV_SKIP_CPU=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-serve > gpurun_out/cab.json 2>/dev/null
  echo "STREAM=$s $(python -c 'import json; d=json.loads(open("gpurun_out/cab.json").read().strip().splitlines()[-1]); print(d["ttft_ms"]["cold_disk"])')"
done
