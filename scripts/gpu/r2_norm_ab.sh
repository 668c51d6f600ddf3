export PYTHONUNBUFFERED=1
for f in 1 0 1; do RDKV_FUSED_NORM=$f RDKV_SKIP_CPU=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-serve --no-extras > gpurun_out/ab_norm_$f.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/ab_norm_$f.json'));k=d['kernels']
print('fused=$f', round(d['ms_per_step'],3), {n:round(k[n]['ms_per_step'],3) for n in ('gemm_qkv','gemm_gate_up','gemm_o','gemm_down','norm_embed','attention')})"; done
timeout 600 python -m pytest tests/test_prefill_gpu.py tests/test_oracle_hf.py tests/test_runtime_gpu.py -m gpu -q -x -p no:cacheprovider --timeout=300 --timeout-method=thread 2>&1 | tail -3
