# stream-K CTA-pair GEMM: correctness under RDKV_GEMM_SK=1/2, then the C3 bench step A/B
for m in 1 2; do
  echo "SK=$m tests: $(RDKV_GEMM_SK=$m timeout 400 python -m pytest tests/test_prefill_gpu.py tests/test_parity_full_gpu.py tests/test_gemm_gpu.py -x -q 2>&1 | tail -1)"
done
for r in 1 2; do
for m in 0 1 2; do
  RDKV_GEMM_SK=$m RDKV_SKIP_CPU=1 timeout 400 python bench.py --steps 10 --warmup 3 --no-serve --no-extras > gpurun_out/sk.json 2>gpurun_out/sk.err
  echo "SK=$m $(python -c 'import json; d=json.loads(open("gpurun_out/sk.json").read().strip().splitlines()[-1]); k=d["kernels"]; print(round(d["value"],1), round(d["ms_per_step"],3), {n: round(k[n]["ms_per_step"],3) for n in ("gemm_qkv","gemm_o","gemm_down","gemm_gate_up")}, d["clocks"]["sm_mhz"])' 2>&1 | tail -1)"
done
done
