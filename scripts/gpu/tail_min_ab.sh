# C2 attention (256 units on 148 SMs): tail split of the last 1.73 waves' units, by minimum tiles per split
for r in 1 2; do
for m in 8 5 4; do
  echo "TAIL_MIN=$m C2 $(RDKV_ATTN_TAIL_MIN=$m python scripts/attn_perf.py --seqs 32 --new 64 --cached 2560 --dh 64 2>&1 | tail -1 | cut -c1-80)"
done
done
for m in 8 4; do
  echo "TAIL_MIN=$m C2 bench $(RDKV_ATTN_TAIL_MIN=$m RDKV_SKIP_CPU=1 timeout 600 python bench.py --model llama-3.2-1b --k 5 --batch 32 --steps 10 --warmup 3 --no-serve --no-extras 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["ms_per_step"],3), round(d["kernels"]["attention"]["ms_per_step"],3), d["clocks"]["sm_mhz"])')"
done
timeout 300 python -m pytest tests/test_attention_gpu.py -x -q 2>&1 | tail -1
RDKV_ATTN_TAIL_MIN=4 timeout 300 python -m pytest tests/test_attention_gpu.py tests/test_prefill_gpu.py -x -q 2>&1 | tail -1
