# A/B of attention variants: correctness of the default build, then attn_perf at C2 / C3 for each lib
set -x
python -m pytest tests/test_attention_gpu.py -x -q 2>&1 | tail -3
for lib in "$@"; do
  for rep in 1 2; do
    RDKV_LIB=$lib python scripts/attn_perf.py --seqs 32 --new 64 --cached 2560 --dh 64 2>&1 | tail -1
    RDKV_LIB=$lib python scripts/attn_perf.py --seqs 16 --new 64 --cached 5120 --dh 128 2>&1 | tail -1
  done
done
