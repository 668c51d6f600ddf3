export PYTHONUNBUFFERED=1 RDKV_SKIP_CPU=1
for cfg in "RDKV_L2_PREFETCH=1 RDKV_GEMM_WPOL=1" "RDKV_L2_PREFETCH=0 RDKV_GEMM_WPOL=0" "RDKV_L2_PREFETCH=1 RDKV_GEMM_WPOL=0" "RDKV_L2_PREFETCH=0 RDKV_GEMM_WPOL=1" "RDKV_L2_PREFETCH=1 RDKV_GEMM_WPOL=1"; do
  env $cfg timeout 600 python bench.py --steps 10 --warmup 3 --no-extras --no-serve > gpurun_out/ab.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);k=d['kernels']
print('$cfg', round(d['value'],1), round(d['ms_per_step'],3), 'prof', round(d['profiled_ms_per_step'],3), {n:round(k[n]['ms_per_step'],3) for n in ('gemm_qkv','attention','gemm_o','gemm_gate_up','gemm_down')}, d['clocks']['sm_mhz'])"
done
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_prefill_gpu.py tests/test_attention_gpu.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
./scripts/micro/mma_rate
