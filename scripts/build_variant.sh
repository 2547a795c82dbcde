#!/bin/bash
# Build an experimental variant of the CUDA library: scripts/build_variant.sh NAME "-DFLAG=..."
set -e
NAME=$1; shift
FLAGS="$*"
SRC=paper_2403_14111_b200/csrc
OUT=/tmp/hcvar_$NAME
mkdir -p $OUT exp
for f in ntt kernels keyswitch context evaluator schedules bootstrap capi; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -Xcompiler -ffp-contract=off -Xcompiler -fno-fast-math --expt-relaxed-constexpr $FLAGS \
    -c $SRC/$f.cu -o $OUT/$f.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o exp/libhc_$NAME.so $OUT/*.o
echo built exp/libhc_$NAME.so
