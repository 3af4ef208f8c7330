#!/bin/bash
# Build a variant libdfm.so with extra -D flags for A/B runs on the GPU box
# (DFM_LIB=build/var_<name>/libdfm.so python bench.py ...):
#   bash tools/build_variant.sh <name> "-DFOO=1 ..." [sources to rebuild, default sortpr_hash]
set -e
NAME=$1; DEFS=$2; SRCS=${3:-sortpr_hash}
OUT=build/var_$NAME; mkdir -p $OUT
ARCH="-gencode arch=compute_100a,code=sm_100a"
OBJS=""
for o in build/*.o; do
  b=$(basename $o .o)
  if [[ " $SRCS " == *" $b "* ]]; then
    nvcc $ARCH -O3 -lineinfo -std=c++17 -Iinclude -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr \
      $DEFS -c paper_2410_22764_b200/csrc/$b.cu -o $OUT/$b.o
    OBJS="$OBJS $OUT/$b.o"
  else
    OBJS="$OBJS $o"
  fi
done
nvcc $ARCH -shared -o $OUT/libdfm.so $OBJS
echo "built $OUT/libdfm.so"
