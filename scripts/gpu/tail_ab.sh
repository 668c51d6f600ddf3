timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q -k "tail or swiglu" 2>&1 | tail -2
for v in 0 1; do
  echo "== RDKV_GEMM_TAIL=$v"
  RDKV_GEMM_TAIL=$v python scripts/gemm_c3.py 2>&1 | grep gate_up | head -2
  RDKV_GEMM_TAIL=$v RDKV_SKIP_CPU=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-extras --no-serve 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', round(d['value'],1), round(d['ms_per_step'],3), {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
done
