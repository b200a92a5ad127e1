#!/bin/bash
# Build only the clock64 tile-trace variant of librsfde.so (tools/tile_trace.py) from the current tree
set -e
cd "$(dirname "$0")/.."
python -m paper_2404_10221_b200.build > /dev/null
OUT=tools/micro/var
mkdir -p $OUT
OBJS=$(ls paper_2404_10221_b200/build/*.o | grep -v pass_L1024.o)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -DRSFDE_TILE_TRACE=1 \
  -I paper_2404_10221_b200/csrc -I include -c paper_2404_10221_b200/csrc/pass_L1024.cu -o $OUT/pass_L1024_trace.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $OUT/librsfde_trace.so $OBJS \
  $OUT/pass_L1024_trace.o -lrt -ldl -lpthread
