#!/bin/bash
# GPU half of tools/tile_variants.sh (the variant libraries are built on the CPU side first):
# launch durations of the C5 K chain for the base build and the RSFDE_TILE_SKIP variants, and the
# per-tile clock64 trace of each of the five tile launches
cd "$(dirname "$0")/.."
for v in base 1 2 3; do
  if [ $v = base ]; then LIB=""; else LIB="--lib tools/micro/var/librsfde_skip$v.so"; fi
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tile_kernel -s 5 -c 5 --csv python tools/prof_kernels.py 511 2 $LIB > gpurun_out/t7_var_$v.csv 2>gpurun_out/t7_var_$v.err
done
for w in 0 1 2 3 4; do python tools/tile_trace.py $w > gpurun_out/t7_trace_$w.txt 2>&1; done
