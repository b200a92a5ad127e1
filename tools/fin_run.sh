#!/bin/bash
# check of the finishing-kernel change: parity (all of test_gpu_parity / test_gpu_shard, the restart / replay / C2 / C3 full-size cases), bench C2 C3 C1
cd "$(dirname "$0")/.."
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -q -x > gpurun_out/fin_parity.log 2>&1; echo "rc $?" >> gpurun_out/fin_parity.log
tail -3 gpurun_out/fin_parity.log
timeout 600 python -m pytest tests/test_gpu_full_size.py -q -x -k "restart or replay or C2 or C3 or x0 or coef" > gpurun_out/fin_parity2.log 2>&1; echo "rc $?" >> gpurun_out/fin_parity2.log
tail -3 gpurun_out/fin_parity2.log
for w in C2 C3 C4; do timeout 300 python bench.py --workload $w --no-cpu-baseline > gpurun_out/fin_bench_$w.json 2> gpurun_out/fin_bench_$w.err; done
