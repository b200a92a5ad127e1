timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_size.py -q -x -k "not C5 and not C4" > gpurun_out/r2d_parity.log 2>&1; echo "rc $?" >> gpurun_out/r2d_parity.log
for w in C3 C2; do timeout 300 python bench.py --workload $w --no-cpu-baseline > gpurun_out/r2d_bench_$w.json 2> gpurun_out/r2d_bench_$w.err; done
