set -x
for w in 0 1 2 3 4; do python tools/tile_trace.py $w > gpurun_out/r2b_trace_$w.txt 2>&1; done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"pass_kernel" -s 3 -c 3 -o gpurun_out/r2b_c3 python tools/prof_kernels.py --cfg C3 2047 2 > gpurun_out/r2b_c3_ncu.log 2>&1
for w in C3 C4 C2; do timeout 300 python bench.py --workload $w --no-cpu-baseline > gpurun_out/r2b_bench_$w.json 2> gpurun_out/r2b_bench_$w.err; done
