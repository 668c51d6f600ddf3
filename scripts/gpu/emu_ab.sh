# exp2 emulation share (of every 8 score groups on the FMA pipe) with the r2s3 schedule
for r in 1 2; do
for v in default 2 4 5; do
  lib=paper_2504_11765_b200/librdkv.so; [ $v != default ] && lib=paper_2504_11765_b200/_variants/librdkv_RDKV_ATTN_EMU_$v.so
  c3=$(RDKV_LIB=$lib python scripts/attn_perf.py --seqs 16 --new 64 --cached 5120 --dh 128 2>&1 | tail -1 | cut -c1-32)
  c2=$(RDKV_LIB=$lib python scripts/attn_perf.py --seqs 32 --new 64 --cached 2560 --dh 64 2>&1 | tail -1 | cut -c1-32)
  echo "EMU=$v C3 $c3 C2 $c2"
done
done
