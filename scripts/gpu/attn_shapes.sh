# attn_perf for each lib over C3, an L2-resident C3-like set, and C2
for lib in "$@"; do
  echo "== $lib"
  for a in "--seqs 16 --new 64 --cached 5120 --dh 128" "--seqs 16 --new 64 --cached 1024 --dh 128" "--seqs 32 --new 64 --cached 2560 --dh 64" "--seqs 32 --new 64 --cached 512 --dh 64"; do
    RDKV_LIB=$lib python scripts/attn_perf.py $a 2>&1 | tail -1 | cut -c1-60
  done
done
