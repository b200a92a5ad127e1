#!/bin/bash
# A/B of the C5 K chain's tile launches on one box: base = tools/micro/var/librsfde_A.so, new = in-tree
# library, alternating (A B A B) to average out drift.  Prints per-launch microseconds.
cd "$(dirname "$0")/.."
for r in 1 2; do
  for v in A B; do
    if [ $v = A ]; then LIB="--lib tools/micro/var/librsfde_A.so"; else LIB=""; fi
    ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tile_kernel -s 5 -c 5 --csv \
      python tools/prof_kernels.py 511 2 $LIB > gpurun_out/ab_${v}_$r.csv 2>/dev/null
  done
done
