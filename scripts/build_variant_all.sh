#!/bin/bash
# Variant of the whole CUDA library with extra -D knobs: scripts/build_variant_all.sh NAME "-DFLAG=..." -> exp/libhc_NAME.so
set -e
NAME=$1; shift
FLAGS="$*"
SRC=paper_2403_14111_b200/csrc
OUT=/tmp/hcvar_$NAME
mkdir -p $OUT exp
for f in ntt kernels keyswitch context evaluator schedules bootstrap capi; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -Xcompiler -ffp-contract=off -Xcompiler -fno-fast-math --expt-relaxed-constexpr -Xptxas -v $FLAGS \
    -c $SRC/$f.cu -o $OUT/$f.o 2> $OUT/$f.ptxas.log &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o exp/libhc_$NAME.so $OUT/*.o
echo built exp/libhc_$NAME.so
