# --set full of the gate/up GEMM: in the C3 step (layer 1's launch) and standalone (random operands)
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:gemm_bf16_tc2 -s 6 -c 1 \
    -o gpurun_out/gateup_step python scripts/prof_step.py --steps 1 > gpurun_out/gateup_step.log 2>&1
echo step_rc=$?
ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_tc2 -s 2 -c 1 \
    -o gpurun_out/gateup_alone python scripts/gemm_one.py 1024 28672 4096 swiglu > gpurun_out/gateup_alone.log 2>&1
echo alone_rc=$?
ls gpurun_out/
