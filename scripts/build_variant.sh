#!/bin/bash
# Build librdkv variants that differ in one compile-time define of one source,
# for on-GPU A/B timing:  scripts/build_variant.sh attention_tc.cu RDKV_ATTN_EMU 0 2 3 4
# -> paper_2504_11765_b200/_variants/librdkv_RDKV_ATTN_EMU_<v>.so  (load with RDKV_LIB=...)
set -e
cd "$(dirname "$0")/.."
python -m paper_2504_11765_b200.build >/dev/null
SRC=$1; DEF=$2; shift 2
OUT=paper_2504_11765_b200/_variants; mkdir -p $OUT
OBJS=$(ls paper_2504_11765_b200/_build/*.o | grep -v "/${SRC}.o")
for v in "$@"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo --expt-relaxed-constexpr -Xcompiler -fPIC \
    -Xcompiler -fvisibility=hidden -DRDKV_BUILD -Iinclude -D$DEF=$v -c paper_2504_11765_b200/csrc/$SRC -o /tmp/var_$v.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/librdkv_${DEF}_$v.so $OBJS /tmp/var_$v.o -lpthread
  echo $OUT/librdkv_${DEF}_$v.so
done
