for v in 0 attn; do
  echo "== RDKV_SMALLM_L2PF=$v"
  RDKV_SMALLM_L2PF=$v bash scripts/gpu/bench_quick.sh 2>&1 | grep -E "^decode|^ttft|^[0-9]" | cut -c1-200
done
