# correctness of the default build, then attn_perf at C3 / C2 for each lib (2 reps)
python -m pytest tests/test_attention_gpu.py -x -q 2>&1 | tail -2
for lib in "$@"; do
  echo "== $lib"
  for rep in 1 2; do
    for a in "--seqs 16 --new 64 --cached 5120 --dh 128" "--seqs 32 --new 64 --cached 2560 --dh 64"; do
      RDKV_LIB=$lib python scripts/attn_perf.py $a 2>&1 | tail -1 | cut -c1-40
    done
  done
done
