# DP + split-tail stream-K (RDKV_GEMM_SK=3): correctness, then the C3 bench step A/B against whole tiles
echo "SK tests: $(timeout 900 python -m pytest tests/test_gemm_sk_gpu.py -x -q 2>&1 | tail -3)"
echo "SK=3 parity: $(RDKV_GEMM_SK=3 timeout 600 python -m pytest tests/test_prefill_gpu.py tests/test_parity_full_gpu.py -x -q 2>&1 | tail -1)"
for r in 1 2 3; do
for v in 0:4 3:4 3:8; do
  m=${v%:*}; sp=${v#*:}
  RDKV_GEMM_SK=$m RDKV_GEMM_SK_SPLIT=$sp RDKV_SKIP_CPU=1 timeout 400 python bench.py --steps 10 --warmup 3 --no-serve --no-extras > gpurun_out/sk.json 2>gpurun_out/sk.err
  echo "SK=$m split=$sp $(python -c 'import json; d=json.loads(open("gpurun_out/sk.json").read().strip().splitlines()[-1]); k=d["kernels"]; print(round(d["value"],1), round(d["ms_per_step"],3), {n: round(k[n]["ms_per_step"],3) for n in ("gemm_qkv","gemm_o","gemm_down","gemm_gate_up")}, d["clocks"]["sm_mhz"])' 2>&1 | tail -1)"
done
done
