#!/bin/bash
# Build a variant of libb2ddp.so for A/B runs: tools/ab_build.sh NAME [SRC_DIR]
# Compiles SRC_DIR/*.cu (default: the package csrc) into tools/ab/NAME/libb2ddp.so.
# Run a tool against it with B2_LIB_PATH=tools/ab/NAME/libb2ddp.so.
# B2_NVCC_EXTRA adds flags, e.g. B2_NVCC_EXTRA=-DB2_DEBUG_BOUNDS for the bounds-checked debug build.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; SRC=${2:-$ROOT/paper_2402_02447_b200/csrc}
OUT=$ROOT/tools/ab/$NAME; mkdir -p $OUT/obj
for f in capi.cu bucket_clip.cu fused_allreduce.cu comm.cu strata.cu presort.cu radix.cu mc.cu draws.cpp; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $B2_NVCC_EXTRA -I$ROOT/include -I$ROOT/paper_2402_02447_b200/csrc \
    -c -o $OUT/obj/$f.o $SRC/$f &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -ldl -lpthread -o $OUT/libb2ddp.so $OUT/obj/*.o
rm -rf $OUT/obj
echo $OUT/libb2ddp.so
