# B-tile TMA multicast across two CTA pairs (RDKV_GEMM_MC): a bounded first run, bit-exactness, parity, then the C3 step A/B
RDKV_GEMM_MC=1 timeout 90 python scripts/gemm_one.py 1024 28672 4096 swiglu > gpurun_out/mc_one.log 2>&1; echo "mc_one rc=$?"; tail -2 gpurun_out/mc_one.log
echo "MC tests: $(timeout 600 python -m pytest tests/test_gemm_sk_gpu.py -x -q -k multicast 2>&1 | tail -2)"
echo "MC fit: $(RDKV_GEMM_MC_VERBOSE=1 RDKV_GEMM_MC=1 timeout 120 python scripts/gemm_one.py 1024 28672 4096 swiglu 2>&1 | grep fit | head -2)"
for r in 1 2; do
for m in 0 1 3; do
  RDKV_GEMM_MC=$m RDKV_SKIP_CPU=1 timeout 400 python bench.py --steps 10 --warmup 3 --no-serve --no-extras > gpurun_out/mc.json 2>gpurun_out/mc.err
  echo "MC=$m $(python -c 'import json; d=json.loads(open("gpurun_out/mc.json").read().strip().splitlines()[-1]); k=d["kernels"]; print(round(d["value"],1), round(d["ms_per_step"],3), {n: round(k[n]["ms_per_step"],3) for n in ("gemm_qkv","gemm_o","gemm_down","gemm_gate_up")}, d["clocks"]["sm_mhz"])' 2>&1 | tail -1)"
done
done
