export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_runtime_gpu.py::test_single_instance_prefetch_and_reuse -m gpu -x -q -p no:cacheprovider --timeout=500 --timeout-method=thread > gpurun_out/rt_fail.txt 2>&1; echo "rt rc=$?"; grep -n "assert\|Error" gpurun_out/rt_fail.txt | head -20
timeout 300 python scripts/micro/nvls_probe.py > gpurun_out/nvls_probe.json 2>&1; cat gpurun_out/nvls_probe.json | tail -3
timeout 600 python scripts/gemm_c3.py > gpurun_out/r2_gemm_c3.txt 2>&1; cat gpurun_out/r2_gemm_c3.txt
RDKV_LIB=paper_2504_11765_b200/_variants/librdkv_RDKV_ATTN_TRACE_1.so timeout 300 python scripts/micro/attn_tile_trace.py --seqs 16 --new 64 --cached 5120 --dh 128 > gpurun_out/attn_trace_c3.txt 2>&1; tail -60 gpurun_out/attn_trace_c3.txt
