# longer interleaved A/B of B-multicast on the multi-wave grid only (RDKV_GEMM_MC=2: gate/up) vs off
for r in 1 2 3 4 5; do
for m in 0 2; do
  RDKV_GEMM_MC=$m RDKV_SKIP_CPU=1 timeout 400 python bench.py --steps 20 --warmup 5 --no-serve --no-extras > gpurun_out/mc.json 2>gpurun_out/mc.err
  echo "MC=$m $(python -c 'import json; d=json.loads(open("gpurun_out/mc.json").read().strip().splitlines()[-1]); k=d["kernels"]; print(round(d["value"],1), round(d["ms_per_step"],3), {n: round(k[n]["ms_per_step"],3) for n in ("gemm_qkv","gemm_o","gemm_down","gemm_gate_up")}, d["clocks"]["sm_mhz"], d["clocks"]["reasons"])' 2>&1 | tail -1)"
done
done
