set -x
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/r2_full_gputest.log 2>&1; echo "rc $?" >> gpurun_out/r2_full_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "rc $?" >> gpurun_out/r2_smoke.log
timeout 600 python bench.py > gpurun_out/r2_bench_C5.json 2> gpurun_out/r2_bench_C5.err
for w in C1 C2 C3 C4; do timeout 300 python bench.py --workload $w > gpurun_out/r2_bench_$w.json 2> gpurun_out/r2_bench_$w.err; done
timeout 300 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/r2_bench_reference.json 2> gpurun_out/r2_bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"tile_kernel" -s 5 -c 5 -o gpurun_out/r2_ncu_tile python tools/prof_kernels.py 511 2 > /dev/null 2>&1
