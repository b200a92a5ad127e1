#!/bin/bash
# C3 check of the in-tree library: parity at the C3 sizes, the C3 / C2 bench lines, one ncu capture of a K chain
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_full_size.py tests/test_gpu_parity.py -q -x -k "C3 or C2 or 2047 or operator or precond" > gpurun_out/c3s_parity.log 2>&1; echo "rc $?" >> gpurun_out/c3s_parity.log
tail -3 gpurun_out/c3s_parity.log
for w in C3 C2; do timeout 300 python bench.py --workload $w --no-cpu-baseline > gpurun_out/c3s_bench_$w.json 2> gpurun_out/c3s_bench_$w.err; done
python tools/prof_kernels.py 2047 20 --cfg C3 > gpurun_out/c3s_prof.txt 2>&1; tail -4 gpurun_out/c3s_prof.txt
ncu --set full --clock-control none --import-source on -k regex:pass_kernel -s 3 -c 3 -f -o gpurun_out/c3s python tools/prof_kernels.py 2047 2 --cfg C3 > gpurun_out/c3s_ncu.log 2>&1
