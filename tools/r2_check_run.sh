set -x
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/r2b_gputest.log 2>&1; echo "rc $?" >> gpurun_out/r2b_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke.log 2>&1; echo "rc $?" >> gpurun_out/r2b_smoke.log
timeout 600 python bench.py > gpurun_out/r2b_bench_C5.json 2> gpurun_out/r2b_bench_C5.err
