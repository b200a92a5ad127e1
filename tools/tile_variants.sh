#!/bin/bash
# Build experiment variants of librsfde.so with parts of the L = 1024 tile pipeline disabled
# (RSFDE_TILE_SKIP: 1 = no FFTs, 2 = no global stores, 3 = neither) into tools/micro/var/, to split
# a pass's time into its compute and memory parts:
#   bash tools/tile_variants.sh && python tools/prof_kernels.py 511 3 --lib tools/micro/var/librsfde_skip1.so
set -e
cd "$(dirname "$0")/.."
python -m paper_2404_10221_b200.build > /dev/null
OUT=tools/micro/var
mkdir -p $OUT
OBJS=$(ls paper_2404_10221_b200/build/*.o | grep -v pass_L1024.o)
for v in 1 2 3; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -DRSFDE_TILE_SKIP=$v \
    -I paper_2404_10221_b200/csrc -I include -c paper_2404_10221_b200/csrc/pass_L1024.cu -o $OUT/pass_L1024_$v.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $OUT/librsfde_skip$v.so $OBJS \
    $OUT/pass_L1024_$v.o -lrt -ldl -lpthread
done
# per-tile clock64 trace variant (tools/tile_trace.py)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -DRSFDE_TILE_TRACE=1 \
  -I paper_2404_10221_b200/csrc -I include -c paper_2404_10221_b200/csrc/pass_L1024.cu -o $OUT/pass_L1024_trace.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $OUT/librsfde_trace.so $OBJS \
  $OUT/pass_L1024_trace.o -lrt -ldl -lpthread
ls $OUT
