#!/bin/bash
# Variant of the CUDA library that differs only in keyswitch.cu's -D knobs:
#   scripts/build_ks_variant.sh NAME "-DFLAG=..."   ->  exp/libhc_NAME.so
# (the other objects come from the default in-tree build; run make first)
set -e
NAME=$1; shift
FLAGS="$*"
SRC=paper_2403_14111_b200/csrc
mkdir -p exp /tmp/hcks_$NAME
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -Xcompiler -ffp-contract=off -Xcompiler -fno-fast-math --expt-relaxed-constexpr -Xptxas -v $FLAGS \
  -c $SRC/keyswitch.cu -o /tmp/hcks_$NAME/keyswitch.o 2> /tmp/hcks_$NAME/ptxas.log
OBJS=$(ls $SRC/build/*.o | grep -v keyswitch.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o exp/libhc_$NAME.so $OBJS /tmp/hcks_$NAME/keyswitch.o
echo built exp/libhc_$NAME.so
