set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2_final_gputest.log 2>&1; echo "rc $?" >> gpurun_out/r2_final_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_final_smoke.log 2>&1; echo "rc $?" >> gpurun_out/r2_final_smoke.log
timeout 600 python bench.py > gpurun_out/r2_final_bench_C5.json 2> gpurun_out/r2_final_bench_C5.err
timeout 300 python bench.py --workload C4 --no-cpu-baseline > gpurun_out/r2_final_bench_C4.json 2> gpurun_out/r2_final_bench_C4.err
