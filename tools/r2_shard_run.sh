timeout 900 python -m pytest tests/test_gpu_shard.py -q -x > gpurun_out/r2c_shard.log 2>&1; echo "rc $?" >> gpurun_out/r2c_shard.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "matvec or precond or tile128 or solve_steps or graph" > gpurun_out/r2c_parity.log 2>&1; echo "rc $?" >> gpurun_out/r2c_parity.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r2c_bench_C5.json 2> gpurun_out/r2c_bench_C5.err
