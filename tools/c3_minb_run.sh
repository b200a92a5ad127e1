#!/bin/bash
# same-box A/B of the C3 (L = 4096) per-pair kernels: A = in-tree library (2 CTAs per SM, 128 registers),
# B = tools/micro/var/librsfde_m3.so (built with -DRSFDE_LAY3_MINB=3: 3 CTAs per SM, 85 registers)
cd "$(dirname "$0")/.."
for r in 1 2; do
  python tools/prof_kernels.py 2047 20 --cfg C3 > gpurun_out/c3ab_A_$r.txt 2>&1
  python tools/prof_kernels.py 2047 20 --cfg C3 --lib tools/micro/var/librsfde_m3.so > gpurun_out/c3ab_B_$r.txt 2>&1
done
timeout 300 python bench.py --workload C3 --no-cpu-baseline > gpurun_out/c3ab_bench_A.json 2> gpurun_out/c3ab_bench_A.err
cp tools/micro/var/librsfde_m3.so paper_2404_10221_b200/librsfde.so
timeout 300 python bench.py --workload C3 --no-cpu-baseline > gpurun_out/c3ab_bench_B.json 2> gpurun_out/c3ab_bench_B.err
timeout 600 python -m pytest tests/test_gpu_full_size.py tests/test_gpu_parity.py -q -x -k "C3 or 2047" > gpurun_out/c3ab_parity_B.log 2>&1; echo "rc $?" >> gpurun_out/c3ab_parity_B.log
tail -n 8 gpurun_out/c3ab_[AB]_*.txt
