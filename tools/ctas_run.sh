# experiment: tile-pass launch durations with 2 and 1 resident CTAs per SM (RSFDE_TILE_CTAS)
for c in 2 1; do
  RSFDE_TILE_CTAS=$c ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tile_kernel -s 5 -c 5 --csv python tools/prof_kernels.py 511 2 > gpurun_out/t10_ctas_$c.csv 2>&1
done
